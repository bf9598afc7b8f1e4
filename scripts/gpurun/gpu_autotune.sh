mkdir -p gpurun_out
for n in 2 8; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n \
    bench.py --gpus $n --share-gpu --try-fused --try-gated --steps 3 --warmup 3 --hidden 1024 --heads 8 --batch 2 --seq 1024 --no-cpu-baseline \
    > gpurun_out/bench_at_$n.json 2> gpurun_out/bench_at_$n.err; echo "rc=$?"; tail -3 gpurun_out/bench_at_$n.err | cut -c1-300
  tail -1 gpurun_out/bench_at_$n.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('N=$n', d['config']['allreduce'], d['config']['launch'], d.get('allreduce_choice'), d['ms_per_step'])"
done
for rep in 1; do python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('N1 ms/step %.4f value %.1f gemm %.1f frac %.3f sm %s'%(d['ms_per_step'],d['value'],r['achieved'],r['frac'],d['clocks']['sm_mhz']))"; done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29544 \
    bench.py --gpus 4 --share-gpu --steps 3 --warmup 3 --hidden 1024 --heads 8 --batch 2 --seq 1024 --no-cpu-baseline \
    > gpurun_out/bench_at_4.json 2> gpurun_out/bench_at_4.err; echo "rc=$?"
tail -1 gpurun_out/bench_at_4.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('N=4 default', d['config']['allreduce'], d['config']['gated'], d['config']['launch'], d.get('allreduce_choice'), d['ms_per_step'])"
