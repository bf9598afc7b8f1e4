# Serpentine-K A/B: parity, per-GEMM DRAM bytes (ncu) with ATP_KSERP=1/0, step time alternating
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider 2>&1 | tail -1
for v in 1 0; do
  ATP_KSERP=$v timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:gemm_sm100 --launch-skip 36 --launch-count 12 --csv --log-file gpurun_out/kserp_dram_$v.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
done
python - <<'PY'
import csv
for v in ('1','0'):
    rows=[r for r in csv.reader(open(f'gpurun_out/kserp_dram_{v}.csv')) if len(r)>10]
    h=rows[0]; mi=h.index('Metric Name'); vi=h.index('Metric Value'); ii=h.index('ID')
    d={}
    for r in rows[1:]:
        d.setdefault(r[ii],{})[r[mi]]=float(r[vi].replace(',',''))
    rd=[x['dram__bytes_read.sum'] for x in d.values()]
    print('KSERP',v,'reads GB',' '.join('%.3f'%(x/1e9 if x>1e6 else x) for x in rd),'sum %.2f'%sum(rd))
PY
for rep in 1 2; do for v in 1 0; do ATP_KSERP=$v python bench.py --steps 100 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('KSERP $v lin ms %.3f value %.1f frac %.3f sm %s'%(d['ms_per_step'],d['value'],r['frac'],d['clocks']['sm_mhz']))"; done; done
for v in 1 0; do ATP_KSERP=$v python bench.py --layer gpt --steps 50 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('KSERP $v gpt ms %.3f value %.1f sm %s'%(d['ms_per_step'],d['value'],d['clocks']['sm_mhz']))"; done
