# Round 2 v7: fused kernel with flat offsets + per-stage empty barriers; emulation repeated (order effects).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_layer.py tests/test_gpu_nccl_multiproc.py -q -p no:cacheprovider -k "fused or nccl or gated" --maxfail=3 > gpurun_out/gpu_v7_tests.log 2>&1; tail -2 gpurun_out/gpu_v7_tests.log
timeout 300 python scripts/trace_step.py --h 5120 --mesh 4x2 --chunks 1,4 --gemm-ctas 132 --fused-ar --ops > gpurun_out/r02_trace_42_fused_v7.txt 2>&1; grep '"mesh"' gpurun_out/r02_trace_42_fused_v7.txt | cut -c1-400
timeout 600 ncu --set full --clock-control none -k regex:fused_ar --launch-skip 64 --launch-count 4 -o gpurun_out/r02_fused_dry_v7 python scripts/trace_step.py --h 5120 --mesh 4x2 --chunks 4 --gemm-ctas 132 --fused-ar > gpurun_out/r02_ncu_fused_v7.log 2>&1; tail -1 gpurun_out/r02_ncu_fused_v7.log
for rep in 1 2; do
  timeout 600 python scripts/emulate_mesh.py --cfg 4 --meshes 4x2,8x1 --chunks 4,1,2 --gemm-ctas 132 >> gpurun_out/r02_emul_v7.jsonl 2>>gpurun_out/r02_emul.err
  timeout 600 python scripts/emulate_mesh.py --cfg 4 --meshes 4x2,8x1 --chunks 1,2,4 --gemm-ctas 132 --fused-ar >> gpurun_out/r02_emul_v7.jsonl 2>>gpurun_out/r02_emul.err
done
cat gpurun_out/r02_emul_v7.jsonl
