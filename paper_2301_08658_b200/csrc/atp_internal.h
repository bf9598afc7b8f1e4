// Internal (non-ABI) declarations shared by the library's translation units.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace atp {

// GEMM epilogue kinds (gemm_sm100.cu).
enum EpiKind : int {
  EPI_BF16 = 0,       // C = bf16(acc + bias)
  EPI_F32 = 1,        // C = fp32(acc + bias)
  EPI_RESID = 2,      // C = bf16(aux + acc + bias)            residual fused (no all-reduce follows)
  EPI_BIAS_GELU = 3,  // C = U = bf16(acc + bias), C2 = H = bf16(GeLU(U))
  EPI_DGELU = 4,      // C = bf16(bf16(acc) * GeLU'(aux))      aux = saved U
};

struct EpiParams {
  void* C = nullptr;
  int64_t ldc = 0;
  const void* bias = nullptr;  // [N] bf16, or nullptr
  const void* aux = nullptr;   // residual (EPI_RESID) or saved U (EPI_DGELU), bf16
  int64_t ldaux = 0;
  void* C2 = nullptr;
  int64_t ldc2 = 0;
};

// Fused GEMM -> reduce-scatter (fused peer-memory all-reduce stages,
// fused_ar.cu): instead of storing its partial sums locally, the epilogue
// stores each 128-row CTA tile with TMA straight into the receive slot of the
// member that owns the tile's row slice (slice j of a chunk = rows
// [k*Mc + j*S, k*Mc + (j+1)*S), S = Mc / p), over NVLink for peers, and
// counts the tile on that member's chunk counter (release, system scope).
constexpr int kMaxPush = 8;
struct PushArgs {
  CUtensorMap tm[kMaxPush];      // member j's receive slot for this rank: [slot rows, N] bf16, 32-row store boxes
  uint32_t* sig[kMaxPush] = {};  // member j's tile counter of this stage's chunk 0
  int p = 0;                     // group size; 0 = ordinary stores into ep.C
  int slice_rows = 0;            // S
};

struct GemmDesc {
  alignas(64) CUtensorMap tmA;
  alignas(64) CUtensorMap tmB;
  alignas(64) CUtensorMap tmC;   // epilogue TMA-store map of ep.C
  alignas(64) CUtensorMap tmC2;  // ... of ep.C2 (EPI_BIAS_GELU), else a copy of tmC
  int M = 0, N = 0, K = 0;
  bool a_mn = false, b_mn = false;
  int bn = 0;        // 128 or 256 (0 = choose)
  int cg = 0;        // 1 = single CTA (128 x bn tile), 2 = CTA pair (256 x bn); 0 = choose
  int max_ctas = 0;  // persistent grid cap (0 = all SMs)
  int group_m = 16;  // M-tiles per raster group (raster_group_m)
  int epi = EPI_BF16;
  EpiParams ep;
  // Chunk signalling (schedule.cpp "signalled stages"): tiles run chunk by
  // chunk (sig_rows rows each) and every CTA-tile of chunk k adds 1 to sig[k]
  // once its output is globally visible.  nullptr = no signalling.
  uint32_t* sig = nullptr;
  int sig_rows = 0;  // rows per chunk: tiles run chunk by chunk (also when only gated)
  // Chunk gating: before loading the A rows of chunk k the producer waits until
  // gate[k] >= gate_target (published by the communication stream once the
  // previous stage's chunk k is all-reduced).  nullptr = no gating.
  const uint32_t* gate = nullptr;
  uint32_t gate_target = 0;
  // Programmatic dependent launch (set by the executor only when the GEMM's
  // sole dependency is the previous kernel of its stream and it spins on no
  // gate: an early-launched CTA must never hold SMs another stream needs).
  bool pdl = false;
  // fused GEMM -> reduce-scatter (push.p > 0; needs sig / sig_rows)
  PushArgs push;
  // fp32 check mode (gemm_f32.cu): dtype 1, raw operands instead of TMA maps
  int dtype = 0;
  const void* A = nullptr;
  const void* B = nullptr;
  int64_t lda = 0, ldb = 0;
};

// C[M,N] = A[M,K] * B[N,K]^T.
//   a_mn == false: A stored row-major [M,K] (pitch lda);  true: A stored [K,M]
//   b_mn == false: B stored row-major [N,K] (pitch ldb);  true: B stored [K,N]
const char* gemm_prepare(GemmDesc& d, const void* A, int64_t lda, bool a_mn, const void* B,
                         int64_t ldb, bool b_mn, int M, int N, int K);
cudaError_t gemm_launch(const GemmDesc& d, cudaStream_t st);
const char* gemm_prepare_f32(GemmDesc& d, const void* A, int64_t lda, bool a_mn, const void* B, int64_t ldb,
                             bool b_mn, int M, int N, int K);
cudaError_t gemm_launch_f32(const GemmDesc& d, cudaStream_t st);
// Tile plan gemm_prepare will use for an M x N output: N tile (128/256) and CTA group (1/2).
void gemm_plan_tile(int M, int N, int* bn, int* cg);
int gemm_tiles(const GemmDesc& d);
int num_sms();
int raster_group_m(int rows_per_mtile, int N, int K);
// 2-D bf16 TMA map over a row-major [rows, cols] matrix (pitch ld elements),
// box [box_rows, box_cols], 128B swizzle, out-of-bounds reads as zero.
bool tmap_bf16_2d(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                  int box_cols);
// Epilogue TMA-store map: [rows, cols] (pitch ld elements of esz bytes), box
// [32 rows][box_cols] with the swizzle of the box row (32 or 64 bytes).
bool make_tmap_out(CUtensorMap* m, const void* ptr, int esz, int64_t rows, int64_t cols, int64_t ld, int box_cols);
// Same for fp32 (box_cols * 4 <= 128 bytes).
bool tmap_f32_2d(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                 int box_cols);

}  // namespace atp
