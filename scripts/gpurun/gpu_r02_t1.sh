mkdir -p gpurun_out
timeout 600 python -m pytest "tests/test_gpu_layer.py::test_layer_fp32_check_mode" -x -q -p no:cacheprovider 2>&1 | tail -40 > gpurun_out/t1_fp32.log
ATP_EW_COMPUTE=0 timeout 600 python -m pytest "tests/test_gpu_layer.py::test_layer_fp32_check_mode" -x -q -p no:cacheprovider 2>&1 | tail -3 >> gpurun_out/t1_fp32.log
timeout 900 python -m pytest tests/test_gpu_layer.py -q -p no:cacheprovider -k "stack or fused" 2>&1 | tail -40 > gpurun_out/t1_new.log
cat gpurun_out/t1_fp32.log | tail -30; tail -30 gpurun_out/t1_new.log
