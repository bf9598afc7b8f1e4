# persistent CLC attention, successor claimed with the item's last load: parity, A/B vs v2
mkdir -p gpurun_out
export ATP_ATTN_FWD=4 ATP_ATTN_BWD=3
timeout 600 python -m pytest tests/test_gpu_attention.py -q -p no:cacheprovider 2>&1 | tail -2
unset ATP_ATTN_FWD ATP_ATTN_BWD
for v in 4 2 4 2; do
  b=2; [ $v = 4 ] && b=3
  ATP_ATTN_FWD=$v ATP_ATTN_BWD=$b timeout 300 python scripts/attn_bench.py > gpurun_out/attn_b_v$v.log 2>&1; echo "fwd v$v bwd v$b"; cut -c1-260 gpurun_out/attn_b_v$v.log
done
