# forward: v4 only for the grouped order (seq <= 4096), v2 for long sequences; parity + bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_gpu_gpt.py -q -p no:cacheprovider 2>&1 | tail -1
for i in 1 2; do timeout 300 python scripts/attn_bench.py 2>&1 | cut -c1-110; done
