# forward v4 with the speculative (running-max) softmax: parity, A/B vs v2
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py -q -p no:cacheprovider 2>&1 | tail -2
for v in 4 2 4 2; do
  ATP_ATTN_FWD=$v timeout 300 python scripts/attn_bench.py > gpurun_out/attn_s_v$v.log 2>&1; echo "fwd v$v"; cut -c1-120 gpurun_out/attn_s_v$v.log
done
