# A/B: L2 evict_first hint on the epilogue TMA stores
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q -p no:cacheprovider 2>&1 | tail -1
for hnt in 0 1; do
  ATP_GEMM_STORE_HINT=$hnt timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_sm100 -c 24 --csv \
    --log-file gpurun_out/hint_$hnt.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  ATP_GEMM_STORE_HINT=$hnt python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('hint=$hnt ms/step %.3f gemm TF/s %.1f sm_mhz %s'%(d['ms_per_step'],r['achieved'],d['clocks']['sm_mhz']))"
done
