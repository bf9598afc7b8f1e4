# compute-sanitizer after the attention backward v2, warp-uniform issue loops, PDL, CUDA graphs, fused LayerNorm
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san2_memcheck_smoke.log 2>&1; tail -2 gpurun_out/san2_memcheck_smoke.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_attention.py -x -q -p no:cacheprovider > gpurun_out/san2_memcheck_attn.log 2>&1; tail -2 gpurun_out/san2_memcheck_attn.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_graph.py -x -q -p no:cacheprovider > gpurun_out/san2_memcheck_gemm_graph.log 2>&1; tail -2 gpurun_out/san2_memcheck_gemm_graph.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_attention.py -x -q -p no:cacheprovider -k "256-128 or 512-256" > gpurun_out/san2_racecheck_attn.log 2>&1; tail -2 gpurun_out/san2_racecheck_attn.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_gemm.py -x -q -p no:cacheprovider -k "not fullsize" > gpurun_out/san2_racecheck_gemm.log 2>&1; tail -2 gpurun_out/san2_racecheck_gemm.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_attention.py tests/test_gpu_gemm.py -x -q -p no:cacheprovider > gpurun_out/san2_synccheck.log 2>&1; tail -2 gpurun_out/san2_synccheck.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_bwd2 -c 1 -o gpurun_out/attn_bwd2_final python scripts/attn_once.py > gpurun_out/attn_ncu_final.log 2>&1; tail -1 gpurun_out/attn_ncu_final.log
