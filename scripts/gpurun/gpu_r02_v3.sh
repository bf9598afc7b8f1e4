# Round 2 v3: two-phase fused kernel (bulk-copy staged), deferred chunk signals, PDL for signalled GEMMs.
mkdir -p gpurun_out
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --share-gpu --steps 3 --warmup 3 --hidden 1024 --heads 8 --batch 2 --seq 1024 --no-cpu-baseline --probe-mib 4"
timeout 400 $B --layers 1 --try-fused > gpurun_out/dbg_n2_fused1.json 2> gpurun_out/dbg_n2_fused1.err; echo "fused L1 rc=$?"; tail -c 400 gpurun_out/dbg_n2_fused1.json
for f in "" "--fused-ar"; do
  timeout 600 python scripts/emulate_mesh.py --cfg 4 --meshes 4x2,8x1,2x4 --chunks 1,2,4 --gemm-ctas 132 $f >> gpurun_out/r02_emul_v3.jsonl 2>>gpurun_out/r02_emul.err
done
cat gpurun_out/r02_emul_v3.jsonl
timeout 300 python scripts/trace_step.py --h 5120 --mesh 4x2 --chunks 1,4 --gemm-ctas 132 --ops > gpurun_out/r02_trace_42_v3.txt 2>&1; grep '"mesh"' gpurun_out/r02_trace_42_v3.txt | cut -c1-500
timeout 300 python scripts/trace_step.py --h 5120 --mesh 4x2 --chunks 4 --gemm-ctas 132 --fused-ar --ops > gpurun_out/r02_trace_42_fused_v3.txt 2>&1; grep '"mesh"' gpurun_out/r02_trace_42_fused_v3.txt | cut -c1-700
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --maxfail=5 > gpurun_out/gpu_all_v3.log 2>&1; tail -5 gpurun_out/gpu_all_v3.log
