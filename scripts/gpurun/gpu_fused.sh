timeout 400 python -m pytest tests/test_gpu_layer.py -x -q -m gpu -p no:cacheprovider -k fused 2>&1 | tail -25
