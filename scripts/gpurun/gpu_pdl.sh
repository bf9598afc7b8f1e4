mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/pdl_tests.log 2>&1; tail -2 gpurun_out/pdl_tests.log
for rep in 1 2 3; do for v in 1 0; do ATP_PDL=$v python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('pdl=$v ms/step %.4f value %.1f sm %s'%(d['ms_per_step'],d['value'],d['clocks']['sm_mhz']))"; done; done
for v in 1 0; do ATP_PDL=$v python bench.py --layer gpt --steps 30 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('gpt pdl=$v ms/step %.4f value %.1f'%(d['ms_per_step'],d['value']))"; done
