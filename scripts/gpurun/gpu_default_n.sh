mkdir -p gpurun_out
for n in 2 8; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2956$n \
    bench.py --gpus $n --share-gpu --steps 3 --warmup 3 --hidden 1024 --heads 8 --batch 2 --seq 1024 --no-cpu-baseline \
    > gpurun_out/bench_def_$n.json 2> gpurun_out/bench_def_$n.err; echo "rc=$?"
  tail -1 gpurun_out/bench_def_$n.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('N=$n', d['config']['allreduce'], d['config']['gated'], d['config']['launch'], d.get('allreduce_choice'), d.get('chunk_choice',{}).get('chosen'), d['gpu_launches'])"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29570 \
    bench.py --gpus 8 --share-gpu --try-gated --steps 3 --warmup 3 --hidden 1024 --heads 8 --batch 2 --seq 1024 --no-cpu-baseline \
    > gpurun_out/bench_tg_8.json 2> gpurun_out/bench_tg_8.err; echo "rc=$?"
tail -1 gpurun_out/bench_tg_8.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('N=8 try-gated', d['config']['allreduce'], d['config']['gated'], d.get('allreduce_choice'))"
