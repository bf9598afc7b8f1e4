# launch list of bench steps (our kernels only) + ncu full of one step (GEMMs + elementwise)
KR='regex:gemm_sm100|gelu_kernel|dgelu_kernel|add_kernel|core_fwd|core_bwd|colsum|group_sum'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" -c 90 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "$KR" -s 54 -c 18 -o gpurun_out/prof_step python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
