"""DRAM traffic of cuBLAS (torch.matmul, bf16) on the h=12288 layer GEMM shapes, for
comparison with libatp's GEMMs under the same ncu metrics (run under ncu):

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:gemm|nvjet|cutlass \
        python scripts/cublas_traffic.py
"""
import torch

h, T = 12288, 8192
F = 4 * h
shapes = {"qkv_fwd": (T, 3 * h, h), "fc2_fwd": (T, h, F), "fc1_fwd": (T, F, h)}
for name, (M, N, K) in shapes.items():
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(K, N, device="cuda").to(torch.bfloat16)
    for _ in range(2):
        C = A @ B
    torch.cuda.synchronize()
    print(name, M, N, K, flush=True)
    del A, B, C
