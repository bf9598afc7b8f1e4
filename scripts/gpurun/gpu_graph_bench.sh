mkdir -p gpurun_out
for rep in 1 2; do
python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_graph.json 2> gpurun_out/bench_graph.err; tail -1 gpurun_out/bench_graph.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('graph   ms/step %.3f value %.1f e2e %.1f launches %d sm %s | %s'%(d['ms_per_step'],d['value'],d['e2e']['value'],d['gpu_launches'],d['clocks']['sm_mhz'],d['config']['launch']))"
python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-graph 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('direct  ms/step %.3f value %.1f e2e %.1f launches %d sm %s | %s'%(d['ms_per_step'],d['value'],d['e2e']['value'],d['gpu_launches'],d['clocks']['sm_mhz'],d['config']['launch']))"
done
python bench.py --layer gpt --steps 30 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('gpt graph ms/step %.3f value %.1f | %s'%(d['ms_per_step'],d['value'],d['config']['launch']))"
timeout 900 python -m pytest tests/test_gpu_nccl_multiproc.py -x -q -p no:cacheprovider > gpurun_out/nccl_mp.log 2>&1; tail -2 gpurun_out/nccl_mp.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 \
    bench.py --gpus 4 --share-gpu --steps 3 --warmup 3 --hidden 1024 --heads 8 --batch 2 --seq 1024 --no-cpu-baseline \
    > gpurun_out/bench_share_4g.json 2> gpurun_out/bench_share_4g.err; echo "rc=$?"; tail -1 gpurun_out/bench_share_4g.json | cut -c1-300; grep -o '"launch": "[^"]*"' gpurun_out/bench_share_4g.json
