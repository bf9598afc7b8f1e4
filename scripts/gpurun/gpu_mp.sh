# Multi-process NCCL data path on one shared GPU (tests + bench at N=2/4/8, --share-gpu).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_nccl_multiproc.py -x -q -p no:cacheprovider > gpurun_out/nccl_mp.log 2>&1; tail -30 gpurun_out/nccl_mp.log
for n in 2 8; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus $n --share-gpu --steps 3 --warmup 3 --hidden 1024 --heads 8 --batch 2 --seq 1024 --no-cpu-baseline \
    > gpurun_out/bench_share_$n.json 2> gpurun_out/bench_share_$n.err; echo "rc=$?"; tail -3 gpurun_out/bench_share_$n.err; cat gpurun_out/bench_share_$n.json
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 \
    bench.py --gpus 4 --share-gpu --layer gpt --steps 3 --warmup 3 --hidden 1024 --heads 8 --batch 2 --seq 1024 --no-cpu-baseline \
    > gpurun_out/bench_share_gpt4.json 2> gpurun_out/bench_share_gpt4.err; echo "rc=$?"; tail -3 gpurun_out/bench_share_gpt4.err; cat gpurun_out/bench_share_gpt4.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29513 \
    bench.py --gpus 8 --share-gpu --fused-ar --gated --probe --steps 3 --warmup 3 --hidden 1024 --heads 8 --batch 2 --seq 1024 --no-cpu-baseline \
    > gpurun_out/bench_share_8f.json 2> gpurun_out/bench_share_8f.err; echo "rc=$?"; tail -3 gpurun_out/bench_share_8f.err; cat gpurun_out/bench_share_8f.json
