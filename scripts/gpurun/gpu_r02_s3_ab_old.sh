# A/B: GEMMs at HEAD vs commit 3576741 (before the die-aware kernel change), same box, alternating; ncu tensor % of the dW GEMM
mkdir -p gpurun_out
for i in 1 2 3; do
  for t in new old; do
    d=.; [ $t = old ] && d=ab_old
    (cd $d && timeout 300 python scripts/gemm_bench.py --h 12288 --no-ref --iters 10 --only fc2_dw,qkv_dw,fc2_fwd,fc1_dx) > gpurun_out/ab_$t.log 2>&1
    echo "$t $(grep -o '"gemm": "[a-z0-9_]*".*"tflops": [0-9.]*' gpurun_out/ab_$t.log | sed 's/"M".*"ms"/ms/' | tr '\n' ' ')"
  done
done
for t in new old; do
  d=.; [ $t = old ] && d=ab_old
  (cd $d && timeout 300 ncu --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,launch__registers_per_thread --clock-control none -k regex:gemm_sm100 --launch-skip 3 --launch-count 1 --csv python scripts/gemm_bench.py --h 12288 --no-ref --iters 1 --only fc2_dw) > gpurun_out/ab_ncu_$t.csv 2>/dev/null
  echo "$t ncu: $(grep -E 'tensor|duration|per_second|registers' gpurun_out/ab_ncu_$t.csv | awk -F'","' '{print $(NF-2)"="$NF}' | tr -d '"' | tr '\n' ' ')"
done
