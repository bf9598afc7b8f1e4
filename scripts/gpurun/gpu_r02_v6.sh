# Round 2 v6: packed-bf16 fused kernel; release-only chunk signals (no fence.sc.sys per warp/tile).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_layer.py tests/test_gpu_graph.py tests/test_gpu_nccl_multiproc.py -q -p no:cacheprovider --maxfail=3 > gpurun_out/gpu_v6_tests.log 2>&1; tail -3 gpurun_out/gpu_v6_tests.log
timeout 300 python scripts/trace_step.py --h 5120 --mesh 4x2 --chunks 1,4 --gemm-ctas 132 --ops > gpurun_out/r02_trace_42_v6.txt 2>&1; grep '"mesh"' gpurun_out/r02_trace_42_v6.txt | cut -c1-400
timeout 300 python scripts/trace_step.py --h 5120 --mesh 4x2 --chunks 1,4 --gemm-ctas 132 --fused-ar --ops > gpurun_out/r02_trace_42_fused_v6.txt 2>&1; grep '"mesh"' gpurun_out/r02_trace_42_fused_v6.txt | cut -c1-400
for f in "" "--fused-ar"; do
  timeout 600 python scripts/emulate_mesh.py --cfg 4 --meshes 4x2,8x1,2x4 --chunks 1,2,4 --gemm-ctas 132 $f >> gpurun_out/r02_emul_v6.jsonl 2>>gpurun_out/r02_emul.err
done
cat gpurun_out/r02_emul_v6.jsonl
timeout 600 ncu --set full --clock-control none -k regex:fused_ar --launch-skip 64 --launch-count 4 -o gpurun_out/r02_fused_dry_v6 python scripts/trace_step.py --h 5120 --mesh 4x2 --chunks 4 --gemm-ctas 132 --fused-ar > gpurun_out/r02_ncu_fused_v6.log 2>&1; tail -1 gpurun_out/r02_ncu_fused_v6.log
