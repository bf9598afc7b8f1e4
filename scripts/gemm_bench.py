"""Time atp_gemm on the layer's GEMM shapes (CUDA events, warm-up, L2-exceeding operands).

    python scripts/gemm_bench.py [--h 4096] [--T 8192] [--d1 1 --d2 1] [--iters 20]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--h", type=int, default=4096)
    p.add_argument("--T", type=int, default=8192)
    p.add_argument("--d1", type=int, default=1)
    p.add_argument("--d2", type=int, default=1)
    p.add_argument("--iters", type=int, default=20)
    p.add_argument("--mode", type=int, default=-1, help="ATP_GEMM_MODE env for the library (-1: leave)")
    p.add_argument("--no-ref", action="store_true", help="skip the cuBLAS reference timing")
    p.add_argument("--only", default="", help="comma-separated GEMM names to run")
    a = p.parse_args()
    import torch
    import paper_2301_08658_b200 as atp

    h, T, d1, d2 = a.h, a.T, a.d1, a.d2
    F = 4 * h
    hc, h1, q1, F1 = h // d2, h // d1, 3 * h // d1, F // d1
    # (name, M, N, K, a_mn, b_mn, f32_out)
    shapes = [
        ("qkv_fwd", T, q1, hc, False, True, False), ("out_fwd", T, hc, h1, False, True, False),
        ("fc1_fwd", T, F1, hc, False, True, False), ("fc2_fwd", T, hc, F1, False, True, False),
        ("fc2_dx", T, F1, hc, False, False, False), ("fc2_dw", F1, hc, T, True, True, True),
        ("fc1_dx", T, hc, F1, False, False, False), ("fc1_dw", hc, F1, T, True, True, True),
        ("out_dx", T, h1, hc, False, False, False), ("out_dw", h1, hc, T, True, True, True),
        ("qkv_dx", T, hc, q1, False, False, False), ("qkv_dw", hc, q1, T, True, True, True),
    ]
    res = []
    tot_fl, tot_ms = 0.0, 0.0
    for name, M, N, K, amn, bmn, f32 in shapes:
        if a.only and name not in a.only.split(","):
            continue
        A = torch.randn((K, M) if amn else (M, K), device="cuda").to(torch.bfloat16)
        B = torch.randn((K, N) if bmn else (N, K), device="cuda").to(torch.bfloat16)
        C = torch.empty((M, N), device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
        for _ in range(3):
            atp.atp_gemm(A, B, C, a_mn=amn, b_mn=bmn)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            atp.atp_gemm(A, B, C, a_mn=amn, b_mn=bmn)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        fl = 2.0 * M * N * K
        tot_fl += fl
        tot_ms += ms
        if a.no_ref:
            res.append({"gemm": name, "M": M, "N": N, "K": K, "ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 1)})
            print(json.dumps(res[-1]), flush=True)
            continue
        # torch reference for context (cuBLAS)
        At = A.t() if amn else A
        Bt = B if bmn else B.t()
        for _ in range(3):
            torch.matmul(At, Bt)
        e0.record()
        for _ in range(a.iters):
            torch.matmul(At, Bt)
        e1.record()
        e1.synchronize()
        ms_ref = e0.elapsed_time(e1) / a.iters
        res.append({"gemm": name, "M": M, "N": N, "K": K, "ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 1),
                    "cublas_tflops": round(fl / ms_ref / 1e9, 1)})
        print(json.dumps(res[-1]), flush=True)
    print(json.dumps({"total_tflops": round(tot_fl / tot_ms / 1e9, 1), "total_ms": round(tot_ms, 3)}))


if __name__ == "__main__":
    main()
