# LayerNorm register-resident row kernels (ATP_LN_ROW=1, default) vs warp-per-row (0): parity, ncu times, GPT bench A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gpt.py tests/test_gpu_gpt_fullsize.py tests/test_gpu_graph.py -x -q -p no:cacheprovider 2>&1 | tail -1
for v in 1 0; do
  ATP_LN_ROW=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k 'regex:ln_(fwd|bwd)' -c 12 --csv \
    --log-file gpurun_out/ln_row_$v.csv python bench.py --layer gpt --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
  python - $v <<'PY'
import csv,collections,sys
rows=[r for r in csv.reader(open(f'gpurun_out/ln_row_{sys.argv[1]}.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value')
agg=collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[1:]: agg[r[ki].split('(')[0]][r[mi]].append(float(r[vi].replace(',','')))
for k,m in agg.items(): print('LN_ROW',sys.argv[1],k,{mm:'%.1f'%(sum(v)/len(v)/1e3) for mm,v in m.items()})
PY
done
for rep in 1 2; do for v in 1 0; do ATP_LN_ROW=$v python bench.py --layer gpt --steps 50 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('LN_ROW $v gpt ms %.3f value %.1f sm %s'%(d['ms_per_step'],d['value'],d['clocks']['sm_mhz']))"; done; done
