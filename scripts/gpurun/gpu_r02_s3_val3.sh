# full -m gpu suite (split-K removed; fused kernels as 2-CTA clusters; fused/gated virtual-mesh tests isolated), smoke
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -q -m gpu -p no:cacheprovider -rw > gpurun_out/gpu_all_s3v3.log 2>&1; echo "suite rc=$?"; tail -3 gpurun_out/gpu_all_s3v3.log
grep -i "timed out\|attempt" gpurun_out/gpu_all_s3v3.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
