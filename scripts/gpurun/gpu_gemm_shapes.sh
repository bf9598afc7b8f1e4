for cfg in "--h 5120 --d1 4 --d2 2" "--h 5120 --d1 8 --d2 1" "--h 4096 --d1 4 --d2 2" "--h 12288 --d1 4 --d2 2"; do
  echo "=== $cfg"; timeout 300 python scripts/gemm_bench.py $cfg --iters 20 2>&1 | tail -13
done
