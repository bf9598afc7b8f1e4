# per-rank compute of the 8-GPU configs with the final session-3 code (collectives elided, GEMM cap 132), alternating order
mkdir -p gpurun_out
for rep in 1 2; do
  timeout 600 python scripts/emulate_mesh.py --cfg 4 --meshes 4x2,8x1 --chunks 1,4 --gemm-ctas 132 >> gpurun_out/r02_emulate_per_rank_s3.jsonl 2>>gpurun_out/emul_s3.err
  timeout 600 python scripts/emulate_mesh.py --cfg 4 --meshes 4x2 --chunks 4,1 --gemm-ctas 132 >> gpurun_out/r02_emulate_per_rank_s3.jsonl 2>>gpurun_out/emul_s3.err
done
timeout 900 python scripts/emulate_mesh.py --layer gpt --cfg 3,4 --meshes 4x2 --chunks 4,1 --gemm-ctas 132 >> gpurun_out/r02_emulate_per_rank_s3.jsonl 2>>gpurun_out/emul_s3.err
cut -c1-150 gpurun_out/r02_emulate_per_rank_s3.jsonl
