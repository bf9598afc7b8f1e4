timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_layer.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -15
ATP_SIGNALLED=0 timeout 600 python -m pytest tests/test_gpu_layer.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -3
timeout 600 python scripts/emulate_mesh.py --cfg 3,4 --meshes 8x1,4x2,2x4 > gpurun_out/emulate2.jsonl 2> gpurun_out/emulate2.err; tail -2 gpurun_out/emulate2.err
cat gpurun_out/emulate2.jsonl
