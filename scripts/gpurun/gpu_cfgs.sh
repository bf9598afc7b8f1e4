mkdir -p gpurun_out
for cfg in "5120 40" "12288 96"; do set -- $cfg
  python bench.py --hidden $1 --heads $2 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_h$1.json 2>/dev/null; tail -1 gpurun_out/bench_h$1.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('h=$1 ms/step %.3f value %.1f gemm TF/s %.1f frac %.3f e2e %.1f sm %s'%(d['ms_per_step'],d['value'],r['achieved'],r['frac'],d['e2e']['value'],d['clocks']['sm_mhz']))"
done
python bench.py --layer gpt --hidden 5120 --heads 40 --steps 20 --no-cpu-baseline > gpurun_out/bench_gpt_h5120.json 2>/dev/null; tail -1 gpurun_out/bench_gpt_h5120.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('gpt h=5120 ms/step %.3f value %.1f attn TF/s %.1f'%(d['ms_per_step'],d['value'],r['attention_tflops']))"
