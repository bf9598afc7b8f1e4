#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace atp {

enum EwKind : int {
  EW_GELU = 0,      // out = GeLU(a)                       [rows, cols]
  EW_DGELU = 1,     // out = out * GeLU'(a)                (in place)
  EW_ADD = 2,       // out = a + out                       (in place)
  EW_CORE_FWD = 3,  // out[rows, cols] = sum_s a[rows, 3*cols] per head
  EW_CORE_BWD = 4,  // out[rows, 3*cols] = expand(a[rows, cols])
  EW_COLSUM = 5,    // out (fp32 [cols]) = column sums of a [rows, cols]
  // full GPT layer (layernorm.cu, attention.cu), bf16 only
  EW_LN_STATS = 6,       // out2 (fp32 [rows][2]) = (sum a, sum a^2) per row
  EW_LN_APPLY = 7,       // out = LN(a) with gamma b, beta c, row sums out2, width n_total; ws = (mean, rstd)
  EW_LN_BWD_STATS = 8,   // out2 = (sum g, sum g*xhat) per row, g = a(dy) * c(gamma), x = b, ws = (mean, rstd)
  EW_LN_BWD_APPLY = 9,   // out = res + rstd * (g - out2_0/n - xhat * out2_1/n)
  EW_LN_PARAM_GRAD = 10, // out = dgamma, res_out = dbeta (fp32 [cols]) over all rows; out2 = workspace
  EW_PACK = 11,          // out [p][rows][cols/p] = a [rows, cols] (pitch lda)
  EW_UNPACK = 12,        // out [rows, cols] (pitch ldo) = a [p][rows][cols/p]
  EW_ATTN_FWD = 13,      // out (ctx, ldo) , out2 (lse) = attention(a = qkv, lda)
  EW_ATTN_BWD = 14,      // out (dqkv, ldo) from a = qkv, b = ctx, res = dctx, out2 = lse, ws = workspace
                         // (EW_ATTN_FWD: optional split-KV scratch ws of n_total bytes)
  // d2 == 1 (the whole row is local, no statistics all-reduce): one kernel per pass
  EW_LN_FWD = 15,        // EW_LN_STATS + EW_LN_APPLY (out2 unused)
  EW_LN_BWD = 16,        // EW_LN_BWD_STATS + EW_LN_BWD_APPLY (out2 unused)
};

struct EwDesc {
  int kind = EW_ADD;
  void* out = nullptr;
  const void* a = nullptr;
  int64_t rows = 0, cols = 0;  // cols: width of `out` (core_fwd) / of `a` (core_bwd, colsum)
  int heads = 1;
  int dtype = 0;  // 0 = bf16, 1 = fp32 (check mode)
  // full-layer kinds (see above)
  const void* b = nullptr;
  const void* c = nullptr;
  const void* res = nullptr;
  void* out2 = nullptr;
  void* ws = nullptr;
  void* res_out = nullptr;
  int64_t lda = 0, ldb = 0, ldo = 0, ldres = 0;  // row pitches (0 = cols)
  int64_t n_total = 0;                           // LayerNorm width over the whole mesh dimension
  int p = 1;                                     // pack / unpack blocks
  int seq = 0, causal = 1;                       // attention
};

constexpr int kMaxGroup = 16;
struct GroupSumArgs {
  void* buf[kMaxGroup];
  int p = 0;
};

cudaError_t ew_launch(const EwDesc& e, cudaStream_t st);
cudaError_t gpt_ew_launch(const EwDesc& e, cudaStream_t st);  // EW_LN_* / EW_PACK / EW_UNPACK
size_t ln_param_workspace_bytes(int64_t cols);
cudaError_t group_sum_launch(const GroupSumArgs& g, int64_t n, int dtype, cudaStream_t st);

}  // namespace atp
