# Same box: in-step GEMM DRAM traffic from ncu --set full vs --metrics (dram only), N=1 bench step h=12288
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-cupti"
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct"
timeout 900 ncu --metrics $M --clock-control none -k regex:gemm_sm100 --launch-skip 36 --launch-count 12 --csv $B > gpurun_out/traffic2_metrics.csv 2>/dev/null
timeout 1200 ncu --set full --clock-control none -k regex:gemm_sm100 --launch-skip 36 --launch-count 12 -o gpurun_out/r02_gemm_full_h12288_v2 $B > gpurun_out/traffic2_full.log 2>&1
tail -1 gpurun_out/traffic2_full.log
timeout 900 ncu --metrics $M --clock-control none -k regex:gemm_sm100 --launch-skip 36 --launch-count 12 --csv $B > gpurun_out/traffic2_metrics_b.csv 2>/dev/null
