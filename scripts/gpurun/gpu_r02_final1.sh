# Round 2 validation: full -m gpu suite, smoke, bench N=1 (default), launch list, GPT bench, reference arm
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_all_f1.log 2>&1; tail -3 gpurun_out/gpu_all_f1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_f1.log 2>&1; tail -2 gpurun_out/smoke_f1.log
timeout 900 python bench.py > gpurun_out/bench_f1.json 2> gpurun_out/bench_f1.err; cut -c1-400 gpurun_out/bench_f1.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:gemm_sm100|colsum|core_|gelu|add_kernel' -c 60 --csv \
  --log-file gpurun_out/r02_launches_h12288.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-cupti > /dev/null 2>&1
timeout 900 python bench.py --layer gpt --steps 30 > gpurun_out/bench_gpt_f1.json 2> gpurun_out/bench_gpt_f1.err; cut -c1-300 gpurun_out/bench_gpt_f1.json
timeout 400 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_f1.json 2> gpurun_out/bench_ref_f1.err; cut -c1-300 gpurun_out/bench_ref_f1.json
