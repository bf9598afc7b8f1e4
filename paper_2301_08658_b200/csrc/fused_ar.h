#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace atp {

constexpr int kSigSlots = 4096;  // per-rank counters per kind (tile, ready, done)
// The tile region splits in two: [0, kGateBase) cumulative tile counters,
// [kGateBase, kSigSlots) chunk gates (written with the call's epoch).
constexpr int kGateBase = kSigSlots / 2;

// One fused all-reduce of one chunk (fused_ar.cu).  The stage's GEMM has
// pushed its partial sums into the members' receive slots (PushArgs): member
// j's region holds p slots [slot_rows, ld] bf16, slot m = sender m, and chunk
// k's slice j lands at slot rows [k*S, (k+1)*S), S = rows / p.
struct FusedArArgs {
  int p = 1, me = 0;                  // group size, my index in the group
  char* peer_base[16] = {};           // members' symmetric buffers (mine at [me])
  int64_t part_off = 0;               // byte offset of the stage's receive region
  int64_t flag_off = 0;               // byte offset of the counters: tile[kSigSlots] ready[..] done[..]
  int64_t ld = 0, width = 0;          // row pitch / valid columns (elements); ld == width
  int64_t row0 = 0, rows = 0;         // the chunk's rows (global row index, count = p * S)
  int64_t chunk = 0, slot_rows = 0;   // chunk index k, rows per sender slot (T / p)
  int sig_slot = 0;
  uint32_t sig_target = 0, ready_target = 0, done_target = 0;
  void* out = nullptr;                // caller's output [T, ld] (gets the all-reduced values)
  int ew_kind = -1;                   // fused elementwise step (EwKind) or -1
  void* ew_out = nullptr;
  const void* ew_a = nullptr;
  int64_t ew_ld = 0, ew_lda = 0, ew_width = 0;
  int64_t head_dim = 0;
  int n_ctas = 16;
};

// Both phases stream through a per-CTA shared-memory ring of kFusedStages
// stages of kFusedStageBytes, filled by 1-D bulk copies (cp.async.bulk): a
// stage holds one piece of each source (phase A: the p partial slots + the
// elementwise step's side input; phase B: the peer's reduced slice + the side
// input).  Bytes in flight per kernel: n_ctas * kFusedStages * kFusedStageBytes
// (32 CTAs: 3 MiB), above both HBM's and NVLink's bandwidth x latency product,
// so neither the local reduction nor the remote pull is latency-bound.
constexpr int kFusedStages = 3;
constexpr int kFusedStageBytes = 32768;
constexpr int kFusedThreads = 512;

cudaError_t fused_ar_launch(const FusedArArgs& a, cudaStream_t st);

}  // namespace atp
