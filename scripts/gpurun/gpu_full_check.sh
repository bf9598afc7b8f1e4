# Full GPU suite + smoke + both bench lines
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/gpu_all.log 2>&1; tail -3 gpurun_out/gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; tail -1 gpurun_out/bench_n1.json
python bench.py --layer gpt --steps 50 > gpurun_out/bench_gpt.json 2> gpurun_out/bench_gpt.err; tail -1 gpurun_out/bench_gpt.json
