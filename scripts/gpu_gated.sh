timeout 600 python -m pytest tests/test_gpu_layer.py -x -q -m gpu -p no:cacheprovider -k "gated or fused or signalled" 2>&1 | tail -4
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider 2>&1 | tail -2
timeout 600 python scripts/emulate_mesh.py --cfg 4 --meshes 8x1,4x2,2x4 --chunks 1,2,4,8 > gpurun_out/emulate5.jsonl 2> gpurun_out/emulate5.err; tail -3 gpurun_out/emulate5.err
ATP_GATED=0 timeout 600 python scripts/emulate_mesh.py --cfg 4 --meshes 4x2 --chunks 2,4 >> gpurun_out/emulate5.jsonl 2>> gpurun_out/emulate5.err
timeout 300 python bench.py --steps 50 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-300
