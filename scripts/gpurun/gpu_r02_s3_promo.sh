# GEMM DRAM traffic vs TMA L2 promotion (h=12288 shapes): ncu dram bytes + time, and event timing
mkdir -p gpurun_out
G="python scripts/gemm_bench.py --h 12288 --no-ref"
for pr in 3 0 2; do
  export ATP_L2PROMO=$pr
  echo "== promo $pr" >> gpurun_out/promo.log
  timeout 300 $G --iters 5 --only fc2_fwd,qkv_fwd,fc2_dw >> gpurun_out/promo.log 2>&1
  for g in fc2_fwd qkv_fwd fc2_dw; do
    timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none \
      -k regex:gemm_sm100 --launch-skip 3 --launch-count 1 --csv $G --iters 1 --only $g > gpurun_out/promo_${pr}_$g.csv 2>/dev/null
    echo "promo $pr $g $(grep -E 'dram__bytes_read|gpu__time|hit_rate|dram__bytes_write' gpurun_out/promo_${pr}_$g.csv | awk -F'","' '{print $(NF-2)"="$NF}' | tr -d '"' | tr '\n' ' ')"
  done
done
unset ATP_L2PROMO
grep -E "==|tflops" gpurun_out/promo.log | cut -c1-200
