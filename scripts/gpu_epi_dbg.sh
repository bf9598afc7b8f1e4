# A/B of the GEMM epilogue cost inside the N=1 layer step: ATP_GEMM_EPI_DBG=0 (normal), 1 (no stores), 2 (no GeLU math), 3 (neither)
mkdir -p gpurun_out
for d in 0 1 2 3; do
  ATP_GEMM_EPI_DBG=$d timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_sm100 -c 24 --csv \
    --log-file gpurun_out/epi_dbg_$d.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  ATP_GEMM_EPI_DBG=$d python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('dbg=$d', 'ms/step %.3f'%d['ms_per_step'], 'gemm TF/s %.1f'%r['achieved'], 'sm_mhz', d['clocks']['sm_mhz'])"
done
