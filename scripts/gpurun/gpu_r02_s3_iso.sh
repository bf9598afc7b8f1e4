timeout 900 python -m pytest tests/test_gpu_layer.py -q -m gpu -p no:cacheprovider -k "fused_push or stack_fused" -rw 2>&1 | tail -2
