mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gpt.py tests/test_gpu_gpt_fullsize.py tests/test_gpu_graph.py -x -q -p no:cacheprovider 2>&1 | tail -1
for rep in 1 2; do python bench.py --layer gpt --steps 50 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('gpt ms/step %.3f value %.1f attn %.1f sm %s'%(d['ms_per_step'],d['value'],r['attention_tflops'],d['clocks']['sm_mhz']))"; done
python scripts/trace_step.py --layer gpt --h 4096 --heads 32 --mesh 1x1 --chunks 1 > gpurun_out/trace_gpt_ln.txt 2>&1; head -1 gpurun_out/trace_gpt_ln.txt | cut -c1-1500
