# Round 2 v4: attention fwd v3 (2 threads / row) vs v2; fused shared-GPU hang localisation; ncu of the fused
# kernels (dry run); graph / layer / multiproc tests.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py -x -q -p no:cacheprovider 2>&1 | tail -3
ATP_ATTN_FWD=2 timeout 300 python scripts/attn_bench.py > gpurun_out/r02_attn_v2.log 2>&1
timeout 300 python scripts/attn_bench.py > gpurun_out/r02_attn_v3.log 2>&1
tail -4 gpurun_out/r02_attn_v2.log; tail -4 gpurun_out/r02_attn_v3.log
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --share-gpu --steps 3 --warmup 3 --hidden 1024 --heads 8 --batch 2 --seq 1024 --no-cpu-baseline --probe-mib 4 --layers 1 --no-baseline --no-e2e"
timeout 200 $B --fused-ar > gpurun_out/dbg_fused_only.json 2> gpurun_out/dbg_fused_only.err; echo "fused-only rc=$?"; grep "\[bench" gpurun_out/dbg_fused_only.err | tail -4
timeout 300 $B --try-fused > gpurun_out/dbg_tryfused.json 2> gpurun_out/dbg_tryfused.err; echo "try-fused rc=$?"; grep "\[bench" gpurun_out/dbg_tryfused.err | tail -6
timeout 600 ncu --set full --clock-control none -k regex:fused_ar --launch-skip 64 --launch-count 4 -o gpurun_out/r02_fused_dry python scripts/trace_step.py --h 5120 --mesh 4x2 --chunks 4 --gemm-ctas 132 --fused-ar > gpurun_out/r02_ncu_fused.log 2>&1; tail -2 gpurun_out/r02_ncu_fused.log
timeout 1500 python -m pytest tests/test_gpu_graph.py tests/test_gpu_layer.py tests/test_gpu_nccl_multiproc.py -q -p no:cacheprovider --maxfail=3 > gpurun_out/gpu_v4_tests.log 2>&1; tail -5 gpurun_out/gpu_v4_tests.log
