# split-KV forward attention on small grids: GPT parity + per-rank GPT trace A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gpt.py tests/test_gpu_attention.py tests/test_gpu_nccl_multiproc.py -q -p no:cacheprovider -k "gpt or attn" 2>&1 | tail -3
for sp in 1 0 1 0; do
  ATP_ATTN_SPLIT=$sp timeout 300 python scripts/trace_step.py --layer gpt --h 5120 --heads 40 --mesh 4x2 --chunks 4 --gemm-ctas 132 > gpurun_out/r02_trace_gpt42_split$sp.txt 2>&1
  python -c "import json;d=json.loads([l for l in open('gpurun_out/r02_trace_gpt42_split$sp.txt') if l.startswith('{')][0]);print('split $sp', d['device_ms_per_call'], d['by_op'].get('s0:attn_fwd'))"
done
timeout 900 python scripts/emulate_mesh.py --layer gpt --cfg 3,4 --meshes 4x2 --chunks 4,2,1 --gemm-ctas 132 > gpurun_out/r02_emul_gpt_split.jsonl 2>&1; cat gpurun_out/r02_emul_gpt_split.jsonl
