# full -m gpu suite (fused/gated virtual-mesh tests isolated in child processes), split-K dW GEMMs; per-rank emulation A/B
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -q -m gpu -p no:cacheprovider -rw > gpurun_out/gpu_all_s3v2.log 2>&1; echo "suite rc=$?"; tail -4 gpurun_out/gpu_all_s3v2.log
grep -i "timed out\|attempt" gpurun_out/gpu_all_s3v2.log | head
for ks in 0 1 0 1; do
  ATP_KSPLIT=$ks timeout 600 python scripts/emulate_mesh.py --cfg 4 --meshes 4x2,8x1 --chunks 1,4 --gemm-ctas 132 > gpurun_out/emul_ks$ks.jsonl 2>>gpurun_out/emul_ks.err
  echo "ksplit env $ks"; cut -c1-140 gpurun_out/emul_ks$ks.jsonl; cat gpurun_out/emul_ks$ks.jsonl >> gpurun_out/emul_ks_all.jsonl
done
