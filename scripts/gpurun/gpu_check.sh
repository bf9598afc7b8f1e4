set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import torch;print(torch.cuda.get_device_name(0))"
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -30
timeout 600 python -m pytest tests/test_gpu_layer.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -40
timeout 120 python __graft_entry__.py smoke
