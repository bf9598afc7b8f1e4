mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_bwd2 -c 1 -o gpurun_out/attn_bwd2 python scripts/attn_once.py > gpurun_out/attn_ncu.log 2>&1
tail -3 gpurun_out/attn_ncu.log
ATP_ATTN_BWD=1 timeout 600 ncu --set full --clock-control none -k regex:attn_bwd_kernel -c 1 -o gpurun_out/attn_bwd1 python scripts/attn_once.py > gpurun_out/attn_ncu1.log 2>&1
tail -3 gpurun_out/attn_ncu1.log
ls -la gpurun_out/*.ncu-rep
