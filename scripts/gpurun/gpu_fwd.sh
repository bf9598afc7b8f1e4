timeout 300 python -m pytest tests/test_gpu_attention.py -x -q -p no:cacheprovider 2>&1 | tail -1; python scripts/attn_bench.py 2>&1 | grep "{" | python -c "
import sys,json
for l in sys.stdin: d=json.loads(l); print(d['b'],d['s'],d['heads'],d['causal'],'fwd',d['fwd_ms'],d['fwd_tflops'],'sdpa',d['sdpa_tflops'],'bwd',d['bwd_ms'],d['bwd_tflops'])"
