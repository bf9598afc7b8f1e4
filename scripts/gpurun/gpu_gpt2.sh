timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:atp -c 200 --csv \
  --log-file gpurun_out/launches_gpt.csv python bench.py --layer gpt --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 python scripts/emulate_mesh.py --layer gpt --cfg 3,4 --meshes 8x1,4x2,2x4 --chunks 1,2,4 --steps 10 > gpurun_out/emu_gpt.jsonl 2> gpurun_out/emu_gpt.err
echo rc=$?
