mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd2 -c 1 -o gpurun_out/attn_fwd2 python scripts/attn_once.py > gpurun_out/attn_fwd_ncu.log 2>&1
tail -1 gpurun_out/attn_fwd_ncu.log
