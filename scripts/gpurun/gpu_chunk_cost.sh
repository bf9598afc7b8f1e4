# Where the chunked (c=4) per-rank compute loses time vs c=1: cfg 4 (4,2), collectives elided.
mkdir -p gpurun_out
python scripts/emulate_mesh.py --cfg 4 --meshes 4x2,8x1 --chunks 1,2,4 --steps 20 > gpurun_out/chunk_cost.jsonl 2> gpurun_out/chunk_cost.err
cat gpurun_out/chunk_cost.jsonl
for c in 1 4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c$c.csv \
    python scripts/emulate_mesh.py --cfg 4 --meshes 4x2 --chunks $c --steps 1 > /dev/null 2>&1
done
ls -la gpurun_out
