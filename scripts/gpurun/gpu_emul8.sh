mkdir -p gpurun_out
python scripts/emulate_mesh.py --cfg 3,4,5 --meshes 8x1,4x2,2x4,1x8 --chunks 1,2,4 --steps 10 > gpurun_out/emul_v8.jsonl 2>&1; grep "^{" gpurun_out/emul_v8.jsonl | wc -l
