# ncu --set full of the persistent attention kernels (fwd v4, bwd v3) at b4 s2048 32 heads causal
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_fwd4|attn_bwd3" -c 2 -o gpurun_out/attn_persist python scripts/attn_once.py > gpurun_out/attn_persist_ncu.log 2>&1
tail -2 gpurun_out/attn_persist_ncu.log
