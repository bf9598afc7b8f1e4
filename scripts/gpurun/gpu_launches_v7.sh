# Launch lists (ncu gpu__time_duration, serialised) of the linear-block and GPT steps, current kernels
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:gemm_sm100|colsum|core_' -c 90 --csv \
  --log-file gpurun_out/launches_v7.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:attn|gemm_sm100|ln_|colsum|block_pack|gelu|core_|add_kernel' -c 200 --csv \
  --log-file gpurun_out/launches_gpt_v7.csv python bench.py --layer gpt --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
ls gpurun_out/launches_*v7.csv
