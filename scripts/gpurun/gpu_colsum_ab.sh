mkdir -p gpurun_out
for rep in 1 2; do
for v in 1 0; do
  ATP_AUX_COLSUM=$v python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('linear aux=$v ms %.3f sm %s'%(d['ms_per_step'],d['clocks']['sm_mhz']))"
  ATP_AUX_COLSUM=$v python bench.py --layer gpt --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('gpt aux=$v ms %.3f sm %s'%(d['ms_per_step'],d['clocks']['sm_mhz']))"
done
done
