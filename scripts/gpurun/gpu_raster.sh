for rep in 1 2; do
for g in default 8 4 0; do
  if [ "$g" = default ]; then unset ATP_GROUP_M; else export ATP_GROUP_M=$g; fi
  timeout 300 python bench.py --steps 100 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import sys, json; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$g', round(d['value'],1), round(d['ms_per_step'],3), 'gemm', round(r['achieved'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
done
