mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_bench.py -q -p no:cacheprovider -k gpt_n2 2>&1 | tail -3
