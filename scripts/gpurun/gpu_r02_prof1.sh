# Round 2: launch list + ncu full GEMM capture of the N=1 bench step (h=12288), per-rank
# emulation of cfg 4 at several GEMM CTA caps, step traces at (4,2) c=1/4.
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-cupti"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/r02_launches_h12288.csv $B > gpurun_out/r02_launch.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:gemm_sm100 --launch-skip 36 --launch-count 12 \
  -o gpurun_out/r02_gemm_full_h12288 $B > gpurun_out/r02_ncufull.log 2>&1
tail -2 gpurun_out/r02_ncufull.log
for cap in 132 140 148; do
  timeout 600 python scripts/emulate_mesh.py --cfg 4 --meshes 4x2,8x1 --chunks 1,2,4 --gemm-ctas $cap >> gpurun_out/r02_emul_caps.jsonl 2>>gpurun_out/r02_emul.err
done
cat gpurun_out/r02_emul_caps.jsonl
for cap in 132 148; do
  timeout 300 python scripts/trace_step.py --h 5120 --mesh 4x2 --chunks 1,4 --gemm-ctas $cap > gpurun_out/r02_trace_42_cap$cap.txt 2>&1
  grep -i "idle\|busy" gpurun_out/r02_trace_42_cap$cap.txt | head -12
done
