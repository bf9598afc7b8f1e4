# Final ncu captures (round 1): one step's 12 GEMMs (--set full), attention fwd/bwd (--set full), launch lists
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_sm100 --launch-skip 36 --launch-count 12 \
  -o gpurun_out/step_gemms_v6 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/ncu_step6.log 2>&1
tail -1 gpurun_out/ncu_step6.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_ -c 4 -o gpurun_out/attn_final python scripts/attn_once.py > gpurun_out/attn_final.log 2>&1
tail -1 gpurun_out/attn_final.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:gemm_sm100|colsum|core_' -c 90 --csv \
  --log-file gpurun_out/launches_v6.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:attn|gemm_sm100|ln_|colsum|block_pack|gelu|core_|add_kernel' -c 200 --csv \
  --log-file gpurun_out/launches_gpt_v6.csv python bench.py --layer gpt --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
ls gpurun_out | tail -5
