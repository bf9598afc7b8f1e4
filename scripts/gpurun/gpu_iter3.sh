timeout 300 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -2
timeout 300 python bench.py --steps 100 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/bench_it.json
python -c "import json;d=json.load(open('gpurun_out/bench_it.json'));print('value',d['value'],'ms',d['ms_per_step'],'gemm',d['roofline']['achieved'],d['roofline']['frac'],d['clocks'])"
KR='regex:gemm_sm100'
timeout 600 ncu --set full --clock-control none -k "$KR" -s 36 -c 12 -o gpurun_out/prof_gemm2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
