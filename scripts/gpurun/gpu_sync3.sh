mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 compute-sanitizer --tool synccheck --print-limit 10 python -m pytest tests/test_gpu_attention.py tests/test_gpu_gemm.py -x -q -p no:cacheprovider > gpurun_out/san3_synccheck.log 2>&1; tail -2 gpurun_out/san3_synccheck.log
ATP_ATTN_BWD=1 ATP_ATTN_FWD=1 timeout 900 compute-sanitizer --tool synccheck --print-limit 10 python -m pytest tests/test_gpu_attention.py -x -q -p no:cacheprovider > gpurun_out/san3_synccheck_v1.log 2>&1; tail -2 gpurun_out/san3_synccheck_v1.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 10 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san3_synccheck_smoke.log 2>&1; tail -2 gpurun_out/san3_synccheck_smoke.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_layer.py -x -q -p no:cacheprovider -k "every_mesh" > gpurun_out/san3_memcheck_layer.log 2>&1; tail -2 gpurun_out/san3_memcheck_layer.log
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_gemm.py tests/test_gpu_layer.py tests/test_gpu_gpt.py -x -q -p no:cacheprovider 2>&1 | tail -1
