// Attention core kernels (attention.cu): internal interface.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace atp {

// nullptr if the shape is supported, else the reason.
const char* attn_check(int64_t T, int64_t seq, int heads, int head_dim, int64_t ld_qkv, int64_t ld_ctx);
// ctx[T, heads*128] (pitch ld_ctx) and lse[heads][T] from qkv[T, 3*heads*128] (pitch ld_qkv).
cudaError_t attn_fwd_launch(const void* qkv, int64_t ld_qkv, int T, int seq, int heads, int causal, void* ctx,
                            int64_t ld_ctx, float* lse, cudaStream_t st);

}  // namespace atp
