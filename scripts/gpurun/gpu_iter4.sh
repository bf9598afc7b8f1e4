timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider 2>&1 | tail -2
timeout 300 python bench.py --steps 100 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_it.json
python -c "import json;d=json.load(open('gpurun_out/bench_it.json'));print('value',d['value'],'ms',d['ms_per_step'],'gemm',d['roofline']['achieved'],d['roofline']['frac'],'ew ms',d['roofline']['elementwise_ms_per_step'],d['clocks'],'e2e',d['e2e']['value'])"
timeout 600 python scripts/emulate_mesh.py --cfg 3,4 --meshes 8x1,4x2,2x4 --fused-ar > gpurun_out/emulate3.jsonl 2> gpurun_out/emulate3.err; tail -3 gpurun_out/emulate3.err
