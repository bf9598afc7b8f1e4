mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_gpt.py tests/test_gpu_gpt_fullsize.py tests/test_gpu_attention.py -x -q -p no:cacheprovider > gpurun_out/gpt_tests.log 2>&1; tail -3 gpurun_out/gpt_tests.log
python bench.py --layer gpt --steps 50 > gpurun_out/bench_gpt.json 2> gpurun_out/bench_gpt.err; tail -1 gpurun_out/bench_gpt.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('gpt ms/step %.3f value %.1f attn_ms %.3f attn TF/s %.1f sm_mhz %s'%(d['ms_per_step'],d['value'],r['attention_ms_per_step'],r['attention_tflops'],d['clocks']['sm_mhz']))"
timeout 300 python scripts/attn_bench.py > gpurun_out/attn_bench_v2.log 2>&1; cat gpurun_out/attn_bench_v2.log
