"""Attention core throughput (fwd, and bwd once it exists) vs torch SDPA on one B200.
FLOPs counted as the work done: causal = 4*d*s(s+1)/2 per head/sequence fwd."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2301_08658_b200 as atp


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    for b, s, heads, causal in [(4, 2048, 32, True), (4, 2048, 40, True), (4, 2048, 32, False), (1, 8192, 8, True)]:
        T = b * s
        qkv = (torch.randn(T, 3 * heads * 128, device="cuda") * 1.5).to(torch.bfloat16)
        ctx = torch.empty(T, heads * 128, device="cuda", dtype=torch.bfloat16)
        lse = torch.empty(heads, T, device="cuda", dtype=torch.float32)
        ms = timeit(lambda: atp.atp_attn_core_fwd(qkv, ctx, lse, s, heads, causal))
        pairs = s * (s + 1) / 2 if causal else s * s
        fl = 4 * 128 * pairs * heads * b
        v = qkv.view(b, s, heads, 3, 128)
        q, k, vv = (v[:, :, :, i].transpose(1, 2) for i in range(3))
        q, k, vv = q.contiguous(), k.contiguous(), vv.contiguous()
        ms_ref = timeit(lambda: torch.nn.functional.scaled_dot_product_attention(q, k, vv, is_causal=causal))
        dctx = torch.randn_like(ctx)
        dqkv = torch.empty_like(qkv)
        ws = torch.empty(atp._abi.lib().atp_attn_core_workspace(T, heads), dtype=torch.uint8, device="cuda")
        atp.atp_attn_core_fwd(qkv, ctx, lse, s, heads, causal)
        msb = timeit(lambda: atp.atp_attn_core_bwd(qkv, ctx, lse, dctx, dqkv, s, heads, causal, ws))
        qg, kg, vg = (t.detach().requires_grad_() for t in (q, k, vv))
        o = torch.nn.functional.scaled_dot_product_attention(qg, kg, vg, is_causal=causal)
        go = torch.randn_like(o)
        msb_ref = timeit(lambda: torch.autograd.grad(o, (qg, kg, vg), go, retain_graph=True))
        print(json.dumps({"b": b, "s": s, "heads": heads, "causal": causal, "fwd_ms": round(ms, 4),
                          "fwd_tflops": round(fl / ms / 1e9, 1), "sdpa_ms": round(ms_ref, 4),
                          "sdpa_tflops": round(fl / ms_ref / 1e9, 1), "bwd_ms": round(msb, 4),
                          "bwd_tflops": round(2.5 * fl / msb / 1e9, 1), "sdpa_bwd_ms": round(msb_ref, 4),
                          "sdpa_bwd_tflops": round(2.5 * fl / msb_ref / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
