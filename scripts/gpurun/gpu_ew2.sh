mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_gemm.py -x -q -p no:cacheprovider > gpurun_out/ew2_tests.log 2>&1; tail -1 gpurun_out/ew2_tests.log
python scripts/trace_step.py --h 5120 --heads 40 --mesh 4x2 --chunks 1,4 > gpurun_out/trace_ew2.jsonl 2>&1
python scripts/emulate_mesh.py --cfg 3,4 --meshes 4x2,8x1 --chunks 1,2,4 --steps 20 > gpurun_out/emul_ew2.jsonl 2>&1; cat gpurun_out/emul_ew2.jsonl
