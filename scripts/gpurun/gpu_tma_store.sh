# TMA-store epilogue: parity, then step time / per-GEMM launch list / per-rank N=8 compute
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/tma_tests.log 2>&1; tail -5 gpurun_out/tma_tests.log
python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_tma.json 2> gpurun_out/bench_tma.err; tail -1 gpurun_out/bench_tma.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('ms/step %.3f value %.1f gemm TF/s %.1f frac %.3f sm_mhz %s e2e %.1f'%(d['ms_per_step'],d['value'],r['achieved'],r['frac'],d['clocks']['sm_mhz'],d['e2e']['value']))"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_sm100 -c 24 --csv \
    --log-file gpurun_out/epi_tma.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python scripts/emulate_mesh.py --cfg 3,4 --meshes 4x2,8x1 --chunks 1,4 --steps 20 > gpurun_out/emul_tma.jsonl 2>&1; cat gpurun_out/emul_tma.jsonl
