# Round 2: full GPU suite after fused v2 (GEMM->RS push + TMA-pull AG), layer stack, ew-on-compute;
# per-rank emulation (NCCL path / fused dry run), bench N=1.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --maxfail=5 > gpurun_out/gpu_all_v2.log 2>&1; tail -8 gpurun_out/gpu_all_v2.log
for f in "" "--fused-ar"; do
  timeout 600 python scripts/emulate_mesh.py --cfg 4 --meshes 4x2,8x1,2x4 --chunks 1,2,4 --gemm-ctas 132 $f >> gpurun_out/r02_emul_v2.jsonl 2>>gpurun_out/r02_emul.err
done
cat gpurun_out/r02_emul_v2.jsonl
timeout 300 python scripts/trace_step.py --h 5120 --mesh 4x2 --chunks 4 --gemm-ctas 132 --fused-ar --ops > gpurun_out/r02_trace_42_fused.txt 2>&1
head -1 gpurun_out/r02_trace_42_fused.txt | cut -c1-900
timeout 900 python bench.py > gpurun_out/bench_v2.json 2> gpurun_out/bench_v2.err; tail -2 gpurun_out/bench_v2.err; cut -c1-600 gpurun_out/bench_v2.json
