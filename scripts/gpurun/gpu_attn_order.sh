mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_gpu_gpt.py -x -q -p no:cacheprovider 2>&1 | tail -1
for o in 0 1; do echo "ATP_ATTN_ORDER=$o"; ATP_ATTN_ORDER=$o python scripts/attn_bench.py 2>&1 | grep "{"; done
