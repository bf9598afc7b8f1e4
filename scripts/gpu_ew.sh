mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_layer.py -x -q -p no:cacheprovider > gpurun_out/ew_tests.log 2>&1; tail -2 gpurun_out/ew_tests.log
python scripts/trace_step.py --h 4096 --heads 32 --mesh 4x2 --chunks 1,4 > gpurun_out/trace_ew.jsonl 2>&1
python scripts/trace_step.py --h 5120 --heads 40 --mesh 4x2 --chunks 1,4 >> gpurun_out/trace_ew.jsonl 2>&1
python scripts/trace_step.py --h 4096 --heads 32 --mesh 4x2 --chunks 4 --ops > gpurun_out/trace_ew_ops.txt 2>&1
python scripts/emulate_mesh.py --cfg 3,4 --meshes 4x2,8x1 --chunks 1,2,4 --steps 20 > gpurun_out/emul_ew.jsonl 2>&1; cat gpurun_out/emul_ew.jsonl
