#pragma once
#include "../../include/atp.h"
#include "runtime.h"

namespace atp {

using LinearFwd = atp_linear_fwd_args;
using LinearBwd = atp_linear_bwd_args;

// Which blocks of one layer to emit into a single chunk pipeline.
struct LayerParts {
  const atp_attn_fwd_args* attn_fwd = nullptr;
  const atp_mlp_fwd_args* mlp_fwd = nullptr;
  const atp_mlp_bwd_args* mlp_bwd = nullptr;
  const atp_attn_bwd_args* attn_bwd = nullptr;
};

// dtype: 0 = bf16 (tcgen05 path), 1 = fp32 check mode
int build_linear_fwd(const RankView& rv, bool colfirst, const LinearFwd& a, int64_t M, int64_t K, int64_t N,
                     int chunks, int dtype, Sched& out);
int build_linear_bwd(const RankView& rv, bool colfirst, const LinearBwd& a, int64_t M, int64_t K, int64_t N,
                     int chunks, int dtype, Sched& out);
int build_layer(const RankView& rv, const LayerParts& p, int64_t T, int64_t h, int64_t F, int64_t heads,
                int chunks, int dtype, Sched& out);
// n layers as one pipeline: forward 0..n-1, backward n-1..0 (parts[l] = layer l).
int build_layer_stack(const RankView& rv, const LayerParts* parts, int n_layers, int64_t T, int64_t h, int64_t F,
                      int64_t heads, int chunks, int dtype, Sched& out);

// Full pre-LN GPT layer: per-rank workspace bytes and schedule.
size_t gpt_workspace_bytes(int d1, int d2, int64_t T, int64_t h, int64_t F, int64_t heads, int64_t seq, int chunks);
int build_gpt_layer(const RankView& rv, const atp_gpt_args& a, int64_t T, int64_t h, int64_t F, int64_t heads,
                    int64_t seq, int chunks, int causal, char* ws, Sched& out);

const char* last_error();
int mesh_create(int d1, int d2, int world_rank, const uint8_t* uid, int device, bool is_virtual, atp_mesh** out);
int mesh_destroy(atp_mesh* m);

}  // namespace atp
