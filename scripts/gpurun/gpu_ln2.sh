# LN parameter-gradient finalize kernel (2D reduce): GPT parity + graph tests, GPT bench, ln_ launch times
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gpt.py tests/test_gpu_gpt_fullsize.py tests/test_gpu_graph.py -x -q -p no:cacheprovider 2>&1 | tail -1
for rep in 1 2; do python bench.py --layer gpt --steps 50 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('gpt ms/step %.3f value %.1f attn %.1f sm %s'%(d['ms_per_step'],d['value'],r['attention_tflops'],d['clocks']['sm_mhz']))"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:ln_' -c 40 --csv \
  --log-file gpurun_out/launches_ln2.csv python bench.py --layer gpt --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
python - <<'PY'
import csv,collections
rows=[r for r in csv.reader(open('gpurun_out/launches_ln2.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
agg=collections.defaultdict(list)
for r in rows[1:]:
    agg[r[ki].split('(')[0]].append(float(r[vi].replace(',','')))
for k,v in agg.items(): print(k, len(v), 'avg us %.1f'%(sum(v)/len(v)/1e3))
PY
