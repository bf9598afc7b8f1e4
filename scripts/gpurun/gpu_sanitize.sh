# compute-sanitizer over small runs of every kernel family (memcheck; initcheck on the GEMM/attention paths)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_memcheck_smoke.log 2>&1; tail -4 gpurun_out/san_memcheck_smoke.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_attention.py -x -q -p no:cacheprovider -k "256-128 or 512-256" > gpurun_out/san_memcheck_attn.log 2>&1; tail -4 gpurun_out/san_memcheck_attn.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_gemm.py -x -q -p no:cacheprovider > gpurun_out/san_memcheck_gemm.log 2>&1; tail -4 gpurun_out/san_memcheck_gemm.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_attention.py -x -q -p no:cacheprovider -k "256-128" > gpurun_out/san_racecheck_attn.log 2>&1; tail -4 gpurun_out/san_racecheck_attn.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_synccheck_smoke.log 2>&1; tail -4 gpurun_out/san_synccheck_smoke.log
