# Round-2 re-entry validation: full -m gpu suite (stop on first failure), smoke, default bench line, GPT bench.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider --maxfail=5 > gpurun_out/gpu_all.log 2>&1; tail -15 gpurun_out/gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -3 gpurun_out/bench_default.err; cut -c1-2500 gpurun_out/bench_default.json
