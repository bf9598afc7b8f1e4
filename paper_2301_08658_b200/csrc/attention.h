// Attention core kernels (attention.cu): internal interface.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace atp {

// nullptr if the shape is supported, else the reason.
const char* attn_check(int64_t T, int64_t seq, int heads, int head_dim, int64_t ld_qkv, int64_t ld_ctx);
// ctx[T, heads*128] (pitch ld_ctx) and lse[heads][T] from qkv[T, 3*heads*128] (pitch ld_qkv).
// ws / ws_bytes (optional): scratch for split-KV on small grids (attn_fwd_split_bytes).
cudaError_t attn_fwd_launch(const void* qkv, int64_t ld_qkv, int T, int seq, int heads, int causal, void* ctx,
                            int64_t ld_ctx, float* lse, cudaStream_t st, void* ws = nullptr, size_t ws_bytes = 0);
// KV splits the forward uses on this shape (1 = none) and the scratch bytes they need.
int attn_fwd_splits(int64_t T, int64_t seq, int heads);
size_t attn_fwd_split_bytes(int64_t T, int64_t seq, int heads);

// Bytes of workspace attn_bwd_launch needs: dQ accumulator [T][heads*128] fp32 + D [heads][T].
size_t attn_workspace_bytes(int64_t T, int heads);
// dqkv[T, 3*heads*128] (pitch ld_dqkv) = d(attention)/d(qkv) for upstream dctx, given the
// forward's qkv, ctx (O) and lse.  Three launches (prep, main, dQ finalize).
cudaError_t attn_bwd_launch(const void* qkv, int64_t ld_qkv, const void* ctx, int64_t ld_ctx, const float* lse,
                            const void* dctx, int64_t ld_dctx, int T, int seq, int heads, int causal, void* dqkv,
                            int64_t ld_dqkv, void* workspace, cudaStream_t st);

}  // namespace atp
