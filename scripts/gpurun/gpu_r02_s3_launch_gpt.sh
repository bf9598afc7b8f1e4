# launch list of the GPT layer step at h=4096 (libatp kernels only) with the persistent attention
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:gemm_sm100|attn|ln_|colsum|core_|gelu|add_kernel|block_pack' -c 120 --csv \
  --log-file gpurun_out/r02_launches_gpt4096.csv python bench.py --layer gpt --hidden 4096 --heads 32 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-cupti > /dev/null 2>&1
echo rc=$?
