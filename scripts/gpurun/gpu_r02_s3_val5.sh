# session-3 closing validation: full -m gpu suite, smoke, bench N=1, GPT bench h=4096
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -q -m gpu -p no:cacheprovider -rw > gpurun_out/gpu_all_s3v5.log 2>&1; echo "suite rc=$?"; tail -2 gpurun_out/gpu_all_s3v5.log
grep -i "timed out\|attempt" gpurun_out/gpu_all_s3v5.log | head -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_s3v5.json 2> gpurun_out/bench_s3v5.err; cut -c1-160 gpurun_out/bench_s3v5.json
timeout 600 python bench.py --layer gpt --hidden 4096 --heads 32 --steps 30 > gpurun_out/bench_gpt4096_s3v5.json 2> gpurun_out/bench_gpt4096_s3v5.err; cut -c1-160 gpurun_out/bench_gpt4096_s3v5.json
