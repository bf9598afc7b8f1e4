# CTA-order chunk width sweep for the persistent attention kernels (b4 s2048 32/40 heads causal + non-causal)
mkdir -p gpurun_out
for rep in 1 2; do
for g in -1 4 8 32; do
  ATP_ATTN_FWD_G=$g ATP_ATTN_BWD_G=$g timeout 300 python scripts/attn_bench.py 2>/dev/null | head -3 | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print('G=$g', d['heads'], d['causal'], d['fwd_ms'], d['bwd_ms'])"
done
done
