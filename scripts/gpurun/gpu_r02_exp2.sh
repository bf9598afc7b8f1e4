# Round 2 experiments: GPT-layer per-rank chunking cost; fused path SM budget (GEMM cap vs fused CTAs)
mkdir -p gpurun_out
timeout 900 python scripts/emulate_mesh.py --layer gpt --cfg 3,4 --meshes 4x2,8x1 --chunks 4,1,2 --gemm-ctas 132 > gpurun_out/r02_emul_gpt.jsonl 2>&1; cat gpurun_out/r02_emul_gpt.jsonl
for cfg in "132 32" "116 64" "100 96"; do
  set -- $cfg
  ATP_FUSED_CTAS=$2 timeout 600 python scripts/emulate_mesh.py --cfg 4 --meshes 4x2 --chunks 4,2 --gemm-ctas $1 --fused-ar >> gpurun_out/r02_emul_fused_budget.jsonl 2>&1
  timeout 600 python scripts/emulate_mesh.py --cfg 4 --meshes 4x2 --chunks 4,2 --gemm-ctas $1 >> gpurun_out/r02_emul_fused_budget.jsonl 2>&1
done
cat gpurun_out/r02_emul_fused_budget.jsonl
