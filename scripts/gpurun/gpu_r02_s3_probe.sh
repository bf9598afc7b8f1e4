# timing probe: forward v4 reading half of S from TMEM (wrong results) vs the real kernel
mkdir -p gpurun_out
for pr in 1 0 1 0; do
  ATP_ATTN_PROBE_HALF_S=$pr timeout 300 python scripts/attn_bench.py > gpurun_out/probe.log 2>&1; echo "half-S probe $pr"; cut -c1-110 gpurun_out/probe.log
done
