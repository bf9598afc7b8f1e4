# virtual mesh: fused CTAs capped at one GPU's budget across ranks: the 32-queue repro and the default, repeated
mkdir -p gpurun_out
for i in 1 2; do
  for c in 32 8; do
    CUDA_DEVICE_MAX_CONNECTIONS=$c ATP_ISOLATED_CHILD=1 timeout 200 python -m pytest "tests/test_gpu_layer.py::test_layer_fused_push_every_stage" "tests/test_gpu_layer.py::test_layer_fused_peer_allreduce" "tests/test_gpu_layer.py::test_layer_chunk_gated" "tests/test_gpu_layer.py::test_layer_stack_fused_and_gated" -q -p no:cacheprovider > gpurun_out/hol3.log 2>&1
    echo "run $i conn $c rc=$? $(tail -1 gpurun_out/hol3.log | cut -c1-70)"
  done
done
