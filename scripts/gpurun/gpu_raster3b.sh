# Parity for the raster rule with the B-fits-L2 case + ncu --set full of one step's 12 GEMMs (traffic v8)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py tests/test_gpu_fullsize.py tests/test_gpu_graph.py -x -q -p no:cacheprovider > gpurun_out/raster3_tests.log 2>&1; tail -1 gpurun_out/raster3_tests.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_sm100 --launch-skip 36 --launch-count 12 \
  -o gpurun_out/step_gemms_v8 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/ncu_step8.log 2>&1
tail -1 gpurun_out/ncu_step8.log
