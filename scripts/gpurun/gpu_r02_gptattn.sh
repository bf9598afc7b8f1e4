# GPT per-rank at c=4: forward attention v1 (one query tile per CTA: 2x the CTAs) vs v2 on small grids
mkdir -p gpurun_out
for v in 2 1 2 1; do
  ATP_ATTN_FWD=$v timeout 300 python scripts/trace_step.py --layer gpt --h 5120 --heads 40 --mesh 4x2 --chunks 4 --gemm-ctas 132 > gpurun_out/r02_trace_gpt42_fwd$v.txt 2>&1
  python -c "import json;d=json.loads([l for l in open('gpurun_out/r02_trace_gpt42_fwd$v.txt') if l.startswith('{')][0]);print('fwd v$v', d['device_ms_per_call'], d['by_op'].get('s0:attn_fwd'))"
done
