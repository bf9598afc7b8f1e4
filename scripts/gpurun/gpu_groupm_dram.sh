# Raster group sweep: per-GEMM DRAM reads (ncu) of one step for fixed ATP_GROUP_M values (serpentine K on)
mkdir -p gpurun_out
for g in 2 4 6 8 12 16 24 32; do
  ATP_GROUP_M=$g timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none \
    -k regex:gemm_sm100 --launch-skip 36 --launch-count 12 --csv --log-file gpurun_out/gm_dram_$g.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
done
python - <<'PY'
import csv
for g in (2,4,6,8,12,16,24,32):
    rows=[r for r in csv.reader(open(f'gpurun_out/gm_dram_{g}.csv')) if len(r)>10]
    h=rows[0]; mi=h.index('Metric Name'); vi=h.index('Metric Value'); ii=h.index('ID')
    d={}
    for r in rows[1:]:
        d.setdefault(r[ii],{})[r[mi]]=float(r[vi].replace(',',''))
    rd=[x['dram__bytes_read.sum'] for x in d.values()]
    us=[x['gpu__time_duration.sum']/1e3 for x in d.values()]
    print('g=%2d'%g,'GB',' '.join('%.3f'%(x/1e9) for x in rd),'sum %.2f'%(sum(rd)/1e9),'| us',' '.join('%.0f'%u for u in us))
PY
