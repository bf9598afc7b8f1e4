timeout 400 python -m pytest tests/test_gpu_layer.py -x -q -m gpu -p no:cacheprovider -k "fused or signalled" 2>&1 | tail -2
for i in 1 2; do
ATP_AUX_COLSUM=0 timeout 300 python bench.py --steps 100 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('aux0 ms',d['ms_per_step'],d['clocks']['sm_mhz'])"
timeout 300 python bench.py --steps 100 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('aux1 ms',d['ms_per_step'],d['clocks']['sm_mhz'])"
done
timeout 600 python scripts/emulate_mesh.py --cfg 4 --meshes 8x1,4x2,2x4 --chunks 1,2,4,8 > gpurun_out/emulate4.jsonl 2> gpurun_out/emulate4.err
timeout 600 python scripts/emulate_mesh.py --cfg 4 --meshes 8x1,4x2,2x4 --chunks 1,2,4,8 --fused-ar >> gpurun_out/emulate4.jsonl 2>> gpurun_out/emulate4.err; tail -3 gpurun_out/emulate4.err
