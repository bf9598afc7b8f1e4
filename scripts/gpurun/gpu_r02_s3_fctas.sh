# fused path dry run (every peer = the rank itself): 16 vs 32 fused CTAs per kernel (2-CTA clusters), cfg 4 (4,2) and (8,1)
mkdir -p gpurun_out
for n in 32 16 32 16; do
  ATP_FUSED_CTAS=$n timeout 600 python scripts/emulate_mesh.py --cfg 4 --meshes 4x2,8x1 --chunks 4,2 --gemm-ctas 132 --fused-ar 2>/dev/null | sed "s/^/ctas $n /" | cut -c1-140
done
