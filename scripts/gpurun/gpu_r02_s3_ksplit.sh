# split-K=2 for the fp32 dW GEMMs on badly quantised grids: parity, per-rank emulation A/B (ATP_KSPLIT=1 = off)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py tests/test_gpu_graph.py tests/test_gpu_fullsize.py -q -p no:cacheprovider 2>&1 | tail -2
for ks in 0 1 0 1; do
  ATP_KSPLIT=$ks timeout 600 python scripts/emulate_mesh.py --cfg 4 --meshes 4x2,8x1 --chunks 1,4 --gemm-ctas 132 > gpurun_out/emul_ks$ks.jsonl 2>>gpurun_out/emul_ks.err
  echo "ksplit env $ks"; cat gpurun_out/emul_ks$ks.jsonl | cut -c1-140
done
