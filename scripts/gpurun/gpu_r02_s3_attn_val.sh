# persistent attention as default: attention + GPT parity suites, smoke, GPT bench at h=4096 (attention share visible) A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_gpt.py tests/test_gpu_gpt_fullsize.py tests/test_gpu_graph.py -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for v in 4 2 4 2; do
  b=3; [ $v = 2 ] && b=2
  ATP_ATTN_FWD=$v ATP_ATTN_BWD=$b timeout 600 python bench.py --layer gpt --hidden 4096 --heads 32 --steps 30 --no-cpu-baseline > gpurun_out/gpt4096_v$v.json 2> gpurun_out/gpt4096_v$v.err
  python -c "import json;d=json.loads(open('gpurun_out/gpt4096_v$v.json').read().strip().splitlines()[-1]);print('v$v', round(d['ms_per_step'],3), round(d['value'],1), d.get('attention_tflops'), d['clocks']['sm_mhz'])"
done
