# Full-layer parity + bench (small, then the default h=4096 shape), plus the linear-block bench.
timeout 600 python -m pytest tests/test_gpu_gpt.py tests/test_gpu_attention.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 300 python bench.py --layer gpt --steps 20 --no-cpu-baseline 2>gpurun_out/gpt_bench.err | tail -1 > gpurun_out/gpt_bench.json
cat gpurun_out/gpt_bench.json
