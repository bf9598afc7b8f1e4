# ncu --set full of one step's 12 GEMM launches (TMA-store epilogue) + attention bwd v2
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_sm100 --launch-skip 36 --launch-count 12 \
  -o gpurun_out/step_gemms_v3 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_step3.log 2>&1
tail -2 gpurun_out/ncu_step3.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_bwd2 -c 1 -o gpurun_out/attn_bwd2_v3 python scripts/attn_once.py > gpurun_out/attn_ncu3.log 2>&1
tail -2 gpurun_out/attn_ncu3.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:attn|gemm_sm100|ln_|colsum|block_pack|gelu|core_|add_kernel' -c 200 --csv \
  --log-file gpurun_out/launches_gpt_v3.csv python bench.py --layer gpt --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:gemm_sm100|colsum|core_' -c 90 --csv \
  --log-file gpurun_out/launches_v3.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out | tail -8
