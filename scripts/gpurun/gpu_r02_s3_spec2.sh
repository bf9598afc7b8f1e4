# forward v4: pipelined speculative softmax (ATP_ATTN_SPEC=1) vs max-first (0) vs v2; parity both ways
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py -q -p no:cacheprovider -k fwd 2>&1 | tail -1
ATP_ATTN_SPEC=0 timeout 600 python -m pytest tests/test_gpu_attention.py -q -p no:cacheprovider -k fwd 2>&1 | tail -1
for cfg in "4 1" "4 0" "2 1" "4 1" "4 0" "2 1"; do
  set -- $cfg
  ATP_ATTN_FWD=$1 ATP_ATTN_SPEC=$2 timeout 300 python scripts/attn_bench.py > gpurun_out/attn_sp.log 2>&1; echo "fwd v$1 spec $2"; cut -c1-100 gpurun_out/attn_sp.log
done
