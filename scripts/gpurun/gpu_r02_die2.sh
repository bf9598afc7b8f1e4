# Die-aware GEMM tile order: parity (GEMM tests), DRAM traffic (ncu) and timing at the h=12288 shapes, bench A/B
mkdir -p gpurun_out
ATP_DIE_AWARE=1 timeout 600 python -m pytest tests/test_gpu_gemm.py -q -p no:cacheprovider 2>&1 | tail -2
G="python scripts/gemm_bench.py --h 12288 --no-ref"
for da in 0 1; do
  export ATP_DIE_AWARE=$da
  for sh in fc2_fwd qkv_fwd fc2_dw; do
    timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_ltcfabric.sum --clock-control none \
      -k regex:gemm_sm100 --launch-skip 3 --launch-count 1 --csv $G --iters 1 --only $sh > gpurun_out/r02_die_ncu_${sh}_da${da}.csv 2>/dev/null
  done
done
for rep in 1 2; do for da in 1 0; do
  echo "== die_aware $da rep $rep" >> gpurun_out/r02_die_gemm.log
  ATP_DIE_AWARE=$da timeout 300 $G --iters 5 >> gpurun_out/r02_die_gemm.log 2>&1
done; done
grep total gpurun_out/r02_die_gemm.log
for da in 1 0 1 0; do
  ATP_DIE_AWARE=$da timeout 600 python bench.py --steps 20 --no-e2e --no-cpu-baseline --no-cupti > gpurun_out/r02_die_bench_$da.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r02_die_bench_$da.json').read().splitlines()[-1]);print('die_aware $da', round(d['ms_per_step'],2), round(d['value'],1), d['clocks']['sm_mhz'])"
done
