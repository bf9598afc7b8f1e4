mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/gelu_tests.log 2>&1; tail -2 gpurun_out/gelu_tests.log
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_sm100 --launch-skip 36 --launch-count 12 --csv \
  --log-file gpurun_out/gelu_epi.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_gelu.json; python -c "
import json; d=json.load(open('gpurun_out/bench_gelu.json')); r=d['roofline']
print('ms/step %.3f value %.1f gemm TF/s %.1f frac %.3f sm_mhz %s'%(d['ms_per_step'],d['value'],r['achieved'],r['frac'],d['clocks']['sm_mhz']))"
