timeout 600 ncu --set full --clock-control none -k regex:gemm_sm100 --launch-skip 36 --launch-count 12 \
  -o gpurun_out/step_gemms_v2 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_step2.log 2>&1
timeout 300 python bench.py --steps 100 2>/dev/null | tail -1 > gpurun_out/b_lin2.json
echo done
