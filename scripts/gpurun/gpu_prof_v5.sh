# ncu --set full of one step's 12 GEMM launches + launch lists + bench lines (after the warp-uniform MMA issue)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_sm100 --launch-skip 36 --launch-count 12 \
  -o gpurun_out/step_gemms_v5 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/ncu_step5.log 2>&1
tail -1 gpurun_out/ncu_step5.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:gemm_sm100|colsum|core_' -c 90 --csv \
  --log-file gpurun_out/launches_v5.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:attn|gemm_sm100|ln_|colsum|block_pack|gelu|core_|add_kernel' -c 200 --csv \
  --log-file gpurun_out/launches_gpt_v5.csv python bench.py --layer gpt --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
python bench.py > gpurun_out/bench_n1_v8.json 2>/dev/null; tail -1 gpurun_out/bench_n1_v8.json | cut -c1-400
python bench.py --layer gpt --steps 50 > gpurun_out/bench_gpt_v6.json 2>/dev/null; tail -1 gpurun_out/bench_gpt_v6.json | cut -c1-400
python scripts/emulate_mesh.py --cfg 3,4 --meshes 8x1,4x2,2x4 --chunks 1,2,4 --steps 20 > gpurun_out/emul_v6.jsonl 2>&1; cat gpurun_out/emul_v6.jsonl
