# Round-end validation: full -m gpu suite, v1 attention kernels, smoke, both bench lines, reference arm
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/gpu_all.log 2>&1; tail -2 gpurun_out/gpu_all.log
ATP_ATTN_BWD=1 ATP_ATTN_FWD=1 timeout 300 python -m pytest tests/test_gpu_attention.py -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -1 gpurun_out/bench_final.json | cut -c1-300
python bench.py --layer gpt --steps 50 > gpurun_out/bench_gpt_final.json 2> gpurun_out/bench_gpt_final.err; tail -1 gpurun_out/bench_gpt_final.json | cut -c1-300
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -1 gpurun_out/bench_ref.json | cut -c1-300
