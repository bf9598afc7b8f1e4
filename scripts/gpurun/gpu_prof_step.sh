# Bench lines (linear block = default, full GPT layer) + ncu captures of one step's GEMMs
# (launch list + --set full for DRAM traffic).  Warm-up: 3 steps x 12 GEMMs = 36 launches skipped.
timeout 300 python bench.py --steps 50 2>gpurun_out/b_lin.err | tail -1 > gpurun_out/b_lin.json
timeout 300 python bench.py --layer gpt --steps 50 2>gpurun_out/b_gpt.err | tail -1 > gpurun_out/b_gpt.json
timeout 600 ncu --set full --clock-control none -k regex:gemm_sm100 --launch-skip 36 --launch-count 12 \
  -o gpurun_out/step_gemms python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_step.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_gpt.csv \
  python bench.py --layer gpt --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo done
