mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py -x -q -p no:cacheprovider > gpurun_out/attn2_tests.log 2>&1; tail -15 gpurun_out/attn2_tests.log
timeout 300 python scripts/attn_bench.py > gpurun_out/attn2_bench.log 2>&1; cat gpurun_out/attn2_bench.log
ATP_ATTN_BWD=1 timeout 300 python scripts/attn_bench.py > gpurun_out/attn1_bench.log 2>&1; cat gpurun_out/attn1_bench.log
