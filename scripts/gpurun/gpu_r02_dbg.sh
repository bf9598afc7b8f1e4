# debug: bench N=2 shared GPU, stack (no fused), then with --try-fused; per-rank emulation after PDL/dedupe
mkdir -p gpurun_out
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --share-gpu --steps 3 --warmup 3 --hidden 1024 --heads 8 --batch 2 --seq 1024 --no-cpu-baseline --probe-mib 4"
timeout 300 $B > gpurun_out/dbg_n2_stack.json 2> gpurun_out/dbg_n2_stack.err; echo "stack rc=$?"; tail -c 600 gpurun_out/dbg_n2_stack.json
timeout 300 $B --layers 1 --try-fused > gpurun_out/dbg_n2_fused1.json 2> gpurun_out/dbg_n2_fused1.err; echo "fused L1 rc=$?"; tail -c 300 gpurun_out/dbg_n2_fused1.json
grep -v "^\[W\|OMP" gpurun_out/dbg_n2_fused1.err | tail -5
timeout 600 python scripts/emulate_mesh.py --cfg 4 --meshes 4x2,8x1 --chunks 1,2,4 --gemm-ctas 132 > gpurun_out/r02_emul_pdl.jsonl 2>&1; cat gpurun_out/r02_emul_pdl.jsonl
timeout 300 python scripts/trace_step.py --h 5120 --mesh 4x2 --chunks 1,4 --gemm-ctas 132 --ops > gpurun_out/r02_trace_42_pdl.txt 2>&1; grep '"mesh"' gpurun_out/r02_trace_42_pdl.txt | cut -c1-700
