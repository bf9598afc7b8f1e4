# LN split kernels with the unrolled column loop: GPT parity, per-rank GPT emulation (4,2) c=4/1, trace
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gpt.py tests/test_gpu_gpt_fullsize.py -q -p no:cacheprovider 2>&1 | tail -1
for rep in 1 2; do timeout 900 python scripts/emulate_mesh.py --layer gpt --cfg 3,4 --meshes 4x2 --chunks 4,1 --gemm-ctas 132 2>/dev/null | cut -c1-120; done
timeout 300 python scripts/trace_step.py --layer gpt --h 5120 --heads 40 --mesh 4x2 --chunks 4 --gemm-ctas 132 > gpurun_out/r02_trace_gpt42_c4_ln.txt 2>&1
python -c "import json;d=json.loads([l for l in open('gpurun_out/r02_trace_gpt42_c4_ln.txt') if l.startswith('{')][0]);print(d['device_ms_per_call'], {k:v for k,v in d['by_op'].items() if 'ln' in k or 'pack' in k})"
