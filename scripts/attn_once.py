"""One forward + backward of the attention core at the N=1 bench shape (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2301_08658_b200 as atp

b, s, heads = 4, 2048, 32
T = b * s
qkv = (torch.randn(T, 3 * heads * 128, device="cuda") * 1.5).to(torch.bfloat16)
ctx = torch.empty(T, heads * 128, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(heads, T, device="cuda", dtype=torch.float32)
dctx = torch.randn_like(ctx)
dqkv = torch.empty_like(qkv)
for _ in range(2):
    atp.atp_attn_core_fwd(qkv, ctx, lse, s, heads, True)
    atp.atp_attn_core_bwd(qkv, ctx, lse, dctx, dqkv, s, heads, True)
torch.cuda.synchronize()
