mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py -x -q -p no:cacheprovider > gpurun_out/attn_tests.log 2>&1; tail -15 gpurun_out/attn_tests.log
timeout 300 python scripts/attn_bench.py 2>&1 | grep -v Warn
timeout 300 python scripts/_attn_trace_tmp.py 2>&1 | head -20
