# Attention forward with paired fp32 softmax ops (FFMA2 / FADD2): parity + bench vs cuDNN
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_gpu_gpt.py -x -q -p no:cacheprovider 2>&1 | tail -1
for rep in 1 2; do python scripts/attn_bench.py 2>&1 | grep "{"; done
