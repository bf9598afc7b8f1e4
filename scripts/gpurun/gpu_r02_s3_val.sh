# Round 2 session 3: validate HEAD (split-KV attention etc.): full -m gpu suite, smoke, bench N=1 default, GPT bench
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_all_s3.log 2>&1; tail -3 gpurun_out/gpu_all_s3.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s3.log 2>&1; tail -2 gpurun_out/smoke_s3.log
timeout 900 python bench.py > gpurun_out/bench_s3.json 2> gpurun_out/bench_s3.err; cut -c1-600 gpurun_out/bench_s3.json
timeout 900 python bench.py --layer gpt --steps 30 > gpurun_out/bench_gpt_s3.json 2> gpurun_out/bench_gpt_s3.err; cut -c1-300 gpurun_out/bench_gpt_s3.json
