# full -m gpu suite after the virtual-mesh fused-CTA budget fix, smoke, bench N=1
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -q -m gpu -p no:cacheprovider -rw > gpurun_out/gpu_all_s3v4.log 2>&1; echo "suite rc=$?"; tail -3 gpurun_out/gpu_all_s3v4.log
grep -i "timed out\|attempt" gpurun_out/gpu_all_s3v4.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_s3v4.json 2> gpurun_out/bench_s3v4.err; cut -c1-200 gpurun_out/bench_s3v4.json
