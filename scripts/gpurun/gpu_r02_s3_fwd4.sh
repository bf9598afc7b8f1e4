# persistent CLC attention (forward v4, backward v3): parity, then A/B vs v2
mkdir -p gpurun_out
export ATP_ATTN_FWD=4 ATP_ATTN_BWD=3
timeout 600 python -m pytest tests/test_gpu_attention.py -q -p no:cacheprovider 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_gpt.py -q -p no:cacheprovider -x 2>&1 | tail -2
unset ATP_ATTN_FWD ATP_ATTN_BWD
for v in 2 4 2 4; do
  b=2; [ $v = 4 ] && b=3
  ATP_ATTN_FWD=$v ATP_ATTN_BWD=$b timeout 300 python scripts/attn_bench.py > gpurun_out/attn_v$v.log 2>&1; echo "fwd v$v bwd v$b"; cut -c1-260 gpurun_out/attn_v$v.log
done
