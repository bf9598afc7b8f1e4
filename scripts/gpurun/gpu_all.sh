timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/gpu_all.log 2>&1; tail -3 gpurun_out/gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:attn|gemm_sm100|ln_|colsum|block_pack|group_sum|gelu|core_|add_kernel' -c 200 --csv \
  --log-file gpurun_out/launches_gpt.csv python bench.py --layer gpt --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo done
