# quick GEMM iteration: parity, per-shape throughput (1-CTA vs 2-CTA), layer parity, bench
timeout 240 python -m pytest tests/test_gpu_gemm.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -15
echo "=== 1-CTA"; ATP_GEMM_MODE=1 timeout 120 python scripts/gemm_bench.py 2>&1 | tail -13
echo "=== default"; timeout 120 python scripts/gemm_bench.py 2>&1 | tail -13
timeout 400 python -m pytest tests/test_gpu_layer.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -5
timeout 300 python bench.py --steps 100 --no-cpu-baseline 2>/dev/null | tail -1
