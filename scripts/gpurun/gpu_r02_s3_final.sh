# Session-3 validation after the persistent attention: full -m gpu suite, smoke, bench N=1 (default), GPT layer
# bench h=4096 and h=12288, GPT launch list (h=4096), reference arm
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_all_s3f.log 2>&1; tail -2 gpurun_out/gpu_all_s3f.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s3f.log 2>&1; tail -2 gpurun_out/smoke_s3f.log
timeout 900 python bench.py > gpurun_out/bench_s3f.json 2> gpurun_out/bench_s3f.err; cut -c1-300 gpurun_out/bench_s3f.json
timeout 900 python bench.py --layer gpt --steps 30 > gpurun_out/bench_gpt_s3f.json 2> gpurun_out/bench_gpt_s3f.err; cut -c1-300 gpurun_out/bench_gpt_s3f.json
timeout 600 python bench.py --layer gpt --hidden 4096 --heads 32 --steps 30 > gpurun_out/bench_gpt4096_s3f.json 2> gpurun_out/bench_gpt4096_s3f.err; cut -c1-300 gpurun_out/bench_gpt4096_s3f.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02_launches_gpt4096.csv \
  python bench.py --layer gpt --hidden 4096 --heads 32 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-cupti > /dev/null 2>&1
timeout 400 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_s3f.json 2> gpurun_out/bench_ref_s3f.err; cut -c1-300 gpurun_out/bench_ref_s3f.json
