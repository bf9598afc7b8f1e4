# head-of-line hypothesis: fused push test (1,8) with 8 vs 32 hardware queues, repeated, in fresh processes
mkdir -p gpurun_out
for i in 1 2 3; do
  for c in 8 32; do
    CUDA_DEVICE_MAX_CONNECTIONS=$c ATP_ISOLATED_CHILD=1 timeout 150 python -m pytest "tests/test_gpu_layer.py::test_layer_fused_push_every_stage[1-8]" "tests/test_gpu_layer.py::test_layer_fused_push_every_stage[4-2]" -q -p no:cacheprovider > gpurun_out/hol.log 2>&1
    echo "run $i conn $c rc=$? $(tail -1 gpurun_out/hol.log | cut -c1-70)"
  done
done
