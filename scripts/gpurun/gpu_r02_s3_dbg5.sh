ATP_ATTN_FWD=5 timeout 100 python /root/repo/scripts/dbg5.py > gpurun_out/dbg5.log 2>&1
grep -c HANG gpurun_out/dbg5.log; grep -v HANG gpurun_out/dbg5.log | tail -3
ATP_ATTN_FWD=5 timeout 300 python -m pytest tests/test_gpu_attention.py -q -p no:cacheprovider -k fwd -x 2>&1 | tail -3
for v in 5 4 5 4; do
  ATP_ATTN_FWD=$v timeout 120 python scripts/attn_bench.py > gpurun_out/attn5_v$v.log 2>&1; echo "fwd v$v"; cut -c1-120 gpurun_out/attn5_v$v.log | grep -v HANG | head -5
done
