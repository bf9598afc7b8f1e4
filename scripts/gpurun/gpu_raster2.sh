# New raster rule + serpentine K: parity, ncu --set full of one step's 12 GEMMs (traffic v7), bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py tests/test_gpu_fullsize.py tests/test_gpu_graph.py -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_sm100 --launch-skip 36 --launch-count 12 \
  -o gpurun_out/step_gemms_v7 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/ncu_step7.log 2>&1
tail -1 gpurun_out/ncu_step7.log
for rep in 1 2; do for g in 0 16; do ATP_GROUP_M=$g python bench.py --steps 100 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('group $g lin ms %.3f value %.1f frac %.3f sm %s'%(d['ms_per_step'],d['value'],r['frac'],d['clocks']['sm_mhz']))"; done; done
python bench.py --layer gpt --steps 50 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/bench_gpt_v11.json
python bench.py > gpurun_out/bench_n1_v13.json 2> gpurun_out/bench_n1_v13.err; tail -c 600 gpurun_out/bench_n1_v13.json
