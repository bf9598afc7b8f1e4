// Local shard GEMM on the 5th-generation tensor cores (sm_100a).
//
// C[M,N] = A[M,K] * B[N,K]^T  (bf16 operands, fp32 accumulation in TMEM)
//
// This is the contraction of every ATP step F3/F6/F8/F11 and of the backward
// products dX = dY W^T and dW = X^T dY (§4.2).  The three
// operand arrangements of the layer map onto the UMMA "major" bits, so no
// operand is ever transposed in HBM:
//     forward   Y  = X  W      A = X  [M,K] K-major,  B = W  [K,N] stored -> MN-major
//     dX        dX = dY W^T    A = dY [M,N] K-major,  B = W  [K,N] stored -> K-major
//     dW        dW = X^T dY    A = X  [T,K] stored -> MN-major, B = dY [T,N] -> MN-major
//
// Design (persistent, warp-specialised, one CTA per SM):
//   warp 0      TMA producer: 128B-swizzled boxes into a STAGES-deep smem ring
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=16)
//   warps 2..9  epilogue: tcgen05.ld -> registers -> fused epilogue -> global
//               (two warps per TMEM lane quadrant, each draining half the columns)
//   TMEM holds two BN-column fp32 accumulators so the epilogue of tile i
//   overlaps the main loop of tile i+1.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <cmath>
#include <mutex>
#include <vector>

#include "atp_internal.h"
#include "gelu.cuh"
#include "sm100_ptx.cuh"

namespace atp {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one swizzle row
constexpr int kEpiWarps = 8;                 // 2 per SM sub-partition: hides epilogue latency
constexpr int kThreads = 64 + 32 * kEpiWarps;  // producer warp + MMA warp + epilogue warps
constexpr uint32_t kBoxBytesMN = 64 * 64 * 2;  // one MN-major box: 64 (mn) x 64 (k)

__device__ __forceinline__ float gelu_f(float x) { return gelu::gelu(x); }
__device__ __forceinline__ float gelu_grad_f(float x) { return gelu::gelu_grad(x); }

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 p = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&p);
}

template <int CG, int BN, int STAGES>
struct SmemLayout {
  static constexpr uint32_t kABytes = BM * BK * 2;             // this CTA's 128 rows of A
  static constexpr uint32_t kBBytes = (BN / CG) * BK * 2;      // this CTA's share of B
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  // epilogue staging: per epilogue warp two 2 KB buffers (double-buffered TMA stores)
  static constexpr uint32_t kStgOffset = STAGES * kStageBytes;
  static constexpr uint32_t kStgBytesPerWarp = 4096;
  static constexpr uint32_t kBarOffset = kStgOffset + kEpiWarps * kStgBytesPerWarp;
  // full[S], empty[S], tmem_full[2], tmem_empty[2], tmem slot
  static constexpr uint32_t kBytes = kBarOffset + (2 * STAGES + 4) * 8 + 16 + 1024;
  static_assert(kBytes <= 232448, "shared memory budget");
};

// Tile order: chunk by chunk (mt_chunk M-tiles per chunk; = all M-tiles when
// not signalling), and inside a chunk groups of kGroupM M-tiles sweep all
// N-tiles, so the ~148 tiles in flight share a few A row-blocks and B
// column-blocks in L2.
__device__ __forceinline__ void tile_coords(int tile, int mt_chunk, int num_n, int group_m, int& mt, int& nt,
                                            int& chunk) {
  const int per_chunk = mt_chunk * num_n;
  chunk = tile / per_chunk;
  const int r0 = tile - chunk * per_chunk;
  const int per_group = group_m * num_n;
  const int g = r0 / per_group;
  const int first = g * group_m;
  const int gm = min(group_m, mt_chunk - first);
  const int r = r0 - g * per_group;
  mt = chunk * mt_chunk + first + r % gm;
  nt = r / gm;
}

// Epilogue slice width: the GeLU / dGeLU / residual epilogues (extra inputs, ~20 FP ops per element)
// so they drain TMEM in 16-column slices to stay within the 168-register budget
// of 320 threads without spilling; the light epilogues use 32-column slices.
template <int EPI>
__host__ __device__ constexpr int slice_width() {
  return EPI == EPI_BF16 ? 32 : 16;
}
// Bytes of one output row of a slice (the TMA store box's inner extent): 64 B
// (SWIZZLE_64B) for bf16 x 32 and fp32 x 16, 32 B (SWIZZLE_32B) for bf16 x 16.
template <int EPI>
__host__ __device__ constexpr int slice_row_bytes() {
  return slice_width<EPI>() * (EPI == EPI_F32 ? 4 : 2);
}
// Swizzled byte offset of 16-byte chunk c of row r (0..31) in a [32 rows][RB bytes]
// staging box: CUTLASS Swizzle<1|2, 4, 3> (the TMA SWIZZLE_32B / _64B patterns),
// which spreads a warp's 32 row-writes over all banks (4 wavefronts per 512 B).
template <int RB>
__device__ __forceinline__ uint32_t stage_off(int r, int c) {
  if constexpr (RB == 64) {
    return static_cast<uint32_t>(r * 64 + ((c ^ ((r >> 1) & 3)) << 4));
  } else {
    return static_cast<uint32_t>(r * 32 + ((c ^ ((r >> 2) & 1)) << 4));
  }
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
template <int EPI>
__host__ __device__ constexpr bool uses_bias() {
  return EPI != EPI_DGELU;
}

// Side inputs of one slice (bias, residual / saved U), fetched as 16-byte
// vectors one slice ahead of their use.
template <int W>
struct Side {
  uint4 bias[W / 8];
  uint4 aux[W / 8];
};

template <int EPI, int W>
__device__ __forceinline__ void load_side(Side<W>& sd, int row, int col0, int M, int N, const EpiParams& ep) {
  const bool in = row < M && col0 < N;
  const bool full = col0 + W <= N;
  if (uses_bias<EPI>() && ep.bias != nullptr) {
    const uint4* b = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(ep.bias) + col0);
#pragma unroll
    for (int g = 0; g < W / 8; ++g)
      sd.bias[g] = (in && (full || col0 + 8 * g + 8 <= N)) ? b[g] : make_uint4(0, 0, 0, 0);
  }
  if constexpr (EPI == EPI_RESID || EPI == EPI_DGELU) {
    const uint4* a = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(ep.aux) +
                                                    static_cast<int64_t>(row) * ep.ldaux + col0);
#pragma unroll
    for (int g = 0; g < W / 8; ++g)
      sd.aux[g] = (in && (full || col0 + 8 * g + 8 <= N)) ? a[g] : make_uint4(0, 0, 0, 0);
  }
}

template <int NV>
__device__ __forceinline__ float bf16_at(const uint4 (&v)[NV], int j) {
  const __nv_bfloat16* p = reinterpret_cast<const __nv_bfloat16*>(&v[j / 8]);
  return __bfloat162float(p[j % 8]);
}

// One W-column slice of one accumulator row (row r = lane of this warp's
// 32-row box): fused epilogue, result written to this warp's shared staging
// box(es) in the swizzled layout the TMA store reads.  Lanes whose row is past
// M still write (the store clips rows >= M and columns >= N).
template <int EPI, int W>
__device__ __forceinline__ void epilogue_chunk(float (&f)[W], const Side<W>& sd, int r, const EpiParams& ep,
                                               uint32_t stg) {
  constexpr int RB = slice_row_bytes<EPI>();
  if (uses_bias<EPI>() && ep.bias != nullptr) {
#pragma unroll
    for (int j = 0; j < W; ++j) f[j] += bf16_at(sd.bias, j);
  }
  if constexpr (EPI == EPI_F32) {
#pragma unroll
    for (int g = 0; g < W / 4; ++g)
      st_shared_v4(stg + stage_off<RB>(r, g), __float_as_uint(f[4 * g]), __float_as_uint(f[4 * g + 1]),
                   __float_as_uint(f[4 * g + 2]), __float_as_uint(f[4 * g + 3]));
  } else {
    if constexpr (EPI == EPI_RESID) {
#pragma unroll
      for (int j = 0; j < W; ++j) f[j] += bf16_at(sd.aux, j);
    }
    if constexpr (EPI == EPI_BIAS_GELU) {
      // U = acc + bias (stored, rounded once); H = GeLU(U) from the rounded U -> second box
      uint32_t hp[W / 2];
#pragma unroll
      for (int j = 0; j < W / 2; ++j) {
        const float u0 = __bfloat162float(__float2bfloat16_rn(f[2 * j]));
        const float u1 = __bfloat162float(__float2bfloat16_rn(f[2 * j + 1]));
        hp[j] = pack_bf16(gelu_f(u0), gelu_f(u1));
      }
#pragma unroll
      for (int g = 0; g < W / 8; ++g)
        st_shared_v4(stg + 32 * RB + stage_off<RB>(r, g), hp[4 * g], hp[4 * g + 1], hp[4 * g + 2], hp[4 * g + 3]);
    }
    if constexpr (EPI == EPI_DGELU) {
      // dU = dH * GeLU'(U); dH is the bf16-rounded product (as after an all-reduce)
#pragma unroll
      for (int j = 0; j < W; ++j) {
        const float dh = __bfloat162float(__float2bfloat16_rn(f[j]));
        f[j] = dh * gelu_grad_f(bf16_at(sd.aux, j));
      }
    }
    uint32_t p[W / 2];
#pragma unroll
    for (int j = 0; j < W / 2; ++j) p[j] = pack_bf16(f[2 * j], f[2 * j + 1]);
#pragma unroll
    for (int g = 0; g < W / 8; ++g)
      st_shared_v4(stg + stage_off<RB>(r, g), p[4 * g], p[4 * g + 1], p[4 * g + 2], p[4 * g + 3]);
  }
}

// CG = 1: one CTA per 128 x BN tile (cta_group::1).
// CG = 2: a CTA pair (cluster of 2) per 256 x BN tile (cta_group::2): each CTA
//         loads its 128 rows of A and BN/2 rows of B, the leader CTA issues
//         M=256 MMAs that read both CTAs' smem, each CTA's TMEM holds its 128
//         accumulator rows; smem stage bytes and L2->SM traffic per FLOP drop
//         by a third.
template <int CG, int BN, int STAGES, int EPI, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_sm100_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmC2,
                      int M, int N, int K, EpiParams ep, uint32_t* sig, int sig_rows, const uint32_t* gate,
                      uint32_t gate_target, int group_m, int kserp, int l2hint,
                      const __grid_constant__ PushArgs push, const uint16_t* die_tab, int dpairs0, int dpairs1) {
  using L = SmemLayout<CG, BN, STAGES>;
  constexpr uint32_t TMEM_COLS = 2 * BN;
  constexpr int BNC = BN / CG;  // B rows loaded by this CTA
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t bar0 = base + L::kBarOffset;
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (STAGES + s); };
  auto tfull_bar = [&](int a) { return bar0 + 8u * (2 * STAGES + a); };
  auto tempty_bar = [&](int a) { return bar0 + 8u * (2 * STAGES + 2 + a); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + L::kBarOffset + (2 * STAGES + 4) * 8);

  const int warp = threadIdx.x / 32;
  const uint32_t lane = threadIdx.x % 32;
  const uint32_t cta_rank = CG == 2 ? ptx::cluster_ctarank() : 0;
  const bool leader = cta_rank == 0;

  const int num_m = (M + BM * CG - 1) / (BM * CG);
  const int num_n = (N + BN - 1) / BN;
  const int num_k = (K + BK - 1) / BK;
  int num_tiles = num_m * num_n;
  int mt_chunk = sig_rows > 0 ? sig_rows / (BM * CG) : num_m;  // M-tiles per chunk
  int unit = blockIdx.x / CG;      // tile-processing unit (CTA or CTA pair)
  int n_units = gridDim.x / CG;
  int m_lo = 0;                    // first M-tile of this unit's tile space
  uint32_t* die_slot = tmem_slot + 1;
  if (die_tab != nullptr && leader && threadIdx.x == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    *die_slot = die_tab[smid];  // broadcast to the peer CTA after the cluster barrier below
  }

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    ptx::prefetch_tmap(&tmC);
    if (EPI == EPI_BIAS_GELU) ptx::prefetch_tmap(&tmC2);
    for (int j = 0; j < push.p; ++j) ptx::prefetch_tmap(&push.tm[j]);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(full_bar(s), 1);
      ptx::mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(tfull_bar(a), 1);
      ptx::mbar_init(tempty_bar(a), kEpiWarps * CG);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (CG == 2) {
      ptx::tmem_alloc_cg2(ptx::smem_u32(tmem_slot), TMEM_COLS);
      ptx::tmem_relinquish_cg2();
    } else {
      ptx::tmem_alloc(ptx::smem_u32(tmem_slot), TMEM_COLS);
      ptx::tmem_relinquish();
    }
  }
  ptx::tc_fence_before();
  if constexpr (CG == 2) {
    ptx::cluster_sync();
  } else {
    __syncthreads();
  }
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (die_tab != nullptr) {
    // Die-aware tiles (ATP_DIE_AWARE; CTA pairs, one CTA per SM, unsignalled):
    // the pairs of each die work on their own share of the M-tiles, so the
    // operand panels a die streams are not fetched into both dies' L2; the
    // pair index within its die comes from the SM -> die table measured at
    // start-up, read by the leader CTA and shared with its peer.
    uint32_t e;
    if (leader) {
      e = *reinterpret_cast<volatile uint32_t*>(die_slot);
    } else {
      asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(e) : "r"(ptx::mapa_shared(ptx::smem_u32(die_slot), 0)));
    }
    const int die = static_cast<int>(e >> 15);
    const int m0 = static_cast<int>((static_cast<int64_t>(num_m) * dpairs0) / (dpairs0 + dpairs1));
    unit = static_cast<int>(e & 0x7fffu);
    n_units = die ? dpairs1 : dpairs0;
    m_lo = die ? m0 : 0;
    mt_chunk = die ? num_m - m0 : m0;
    num_tiles = mt_chunk * num_n;
  }
  // Programmatic dependent launch: the set-up above (barriers, TMEM, tensor-map
  // prefetch) overlapped the previous kernel's tail; the next GEMM may now be
  // scheduled onto SMs as this grid's CTAs retire, and nothing here touches
  // global memory before the previous grid has completed and flushed.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0) {
    {
      // ------------------------------------------------ TMA producer (both CTAs)
      // whole warp runs the loop; one elected lane issues each TMA / expect_tx
      int stage = 0;
      uint32_t phase = 0;
      int gated_chunk = -1;
      // L2 policies (ATP_L2HINT bits): 1 = A evict_last, 2 = B evict_first, 4 = B evict_last
      const uint64_t pol_last = ptx::policy_evict_last(), pol_first = ptx::policy_evict_first();
      const bool hint_a = l2hint & 1, hint_b = l2hint & 6;
      const uint64_t pol_b = (l2hint & 4) ? pol_last : pol_first;
      for (int tile = unit; tile < num_tiles; tile += n_units) {
        int mt, nt, chunk;
        tile_coords(tile, mt_chunk, num_n, group_m, mt, nt, chunk);
        mt += m_lo;
        const int m0 = mt * BM * CG + BM * static_cast<int>(cta_rank);
        const int nb = nt * BN + BNC * static_cast<int>(cta_rank);
        if (gate != nullptr && chunk > gated_chunk) {  // tiles are chunk-major: chunk only grows
          ptx::wait_flag_geq(gate + chunk, gate_target);
          gated_chunk = chunk;
        }
        // serpentine K: odd persistent rounds walk K backwards, so a round
        // starts on the K-blocks the previous round (same A or B panels under
        // the raster) touched last, which are still in L2
        const bool k_rev = kserp && ((tile / n_units) & 1);
        for (int kb = 0; kb < num_k; ++kb) {
          ptx::mbar_wait(empty_bar(stage), phase ^ 1);
          const uint32_t sA = base + stage * L::kStageBytes;
          const uint32_t sB = sA + L::kABytes;
          const uint32_t fb = full_bar(stage);
          if (leader) ptx::mbar_arrive_expect_tx_w(fb, L::kStageBytes * CG);
          const int k0 = (k_rev ? num_k - 1 - kb : kb) * BK;
          auto load = [&](uint32_t dst, const CUtensorMap* tm, int c0, int c1, bool hint, uint64_t pol) {
            if constexpr (CG == 2) {
              if (hint) ptx::tma_load_2d_cg2_hint_w(dst, tm, fb, c0, c1, pol);
              else ptx::tma_load_2d_cg2_w(dst, tm, fb, c0, c1);
            } else {
              if (hint) ptx::tma_load_2d_hint_w(dst, tm, fb, c0, c1, pol);
              else ptx::tma_load_2d_w(dst, tm, fb, c0, c1);
            }
          };
          if constexpr (!A_MN) {
            load(sA, &tmA, k0, m0, hint_a, pol_last);
          } else {
            load(sA, &tmA, m0, k0, hint_a, pol_last);
            load(sA + kBoxBytesMN, &tmA, m0 + 64, k0, hint_a, pol_last);
          }
          if constexpr (!B_MN) {
            load(sB, &tmB, k0, nb, hint_b, pol_b);
          } else {
#pragma unroll
            for (int j = 0; j < BNC / 64; ++j) load(sB + j * kBoxBytesMN, &tmB, nb + 64 * j, k0, hint_b, pol_b);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      // producer tail: wait until the MMA has released every stage (each
      // mbarrier phase gets a waiter; synccheck-clean, no early exit with
      // stages still being read)
      for (int i = 0; i < STAGES; ++i) {
        ptx::mbar_wait(empty_bar(stage), phase ^ 1);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ------------------------------------------------ MMA issuer (leader CTA only)
      // The whole warp runs the loop and one elected lane issues each tcgen05
      // op; the stage descriptors are built once and advanced by constants, so
      // the issue cost per MMA is a few uniform instructions even while the
      // epilogue warps of the same sub-partitions are busy.
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(BM * CG, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
      auto adv = [](uint64_t d, uint32_t bytes) { return d + (bytes >> 4); };
      const uint64_t a0 = A_MN ? ptx::smem_desc_sw128(base, kBoxBytesMN, 1024) : ptx::smem_desc_sw128(base, 16, 1024);
      const uint64_t b0 = B_MN ? ptx::smem_desc_sw128(base + L::kABytes, kBoxBytesMN, 1024)
                               : ptx::smem_desc_sw128(base + L::kABytes, 16, 1024);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = unit; tile < num_tiles; tile += n_units) {
        ptx::mbar_wait(tempty_bar(acc), acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_k; ++kb) {
          ptx::mbar_wait(full_bar(stage), phase);
          ptx::tc_fence_after();
          const uint32_t so = static_cast<uint32_t>(stage) * L::kStageBytes;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = adv(a0, so + (A_MN ? kk * 2048 : kk * 32));
            const uint64_t bd = adv(b0, so + (B_MN ? kk * 2048 : kk * 32));
            if constexpr (CG == 2) {
              ptx::mma_bf16_ss_cg2_w(d_tmem, ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
            } else {
              ptx::mma_bf16_ss_w(d_tmem, ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
            }
          }
          if constexpr (CG == 2) {
            ptx::mma_commit_cg2_mc_w(empty_bar(stage), 0x3);
          } else {
            ptx::mma_commit_w(empty_bar(stage));
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (CG == 2) {
          ptx::mma_commit_cg2_mc_w(tfull_bar(acc), 0x3);
        } else {
          ptx::mma_commit_w(tfull_bar(acc));
        }
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      // tail: both accumulators drained by the epilogue (every phase waited)
      for (int i = 0; i < 2; ++i) {
        ptx::mbar_wait(tempty_bar(acc), acc_phase ^ 1);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ------------------------------------------------ epilogue warps 2..9 (both CTAs)
    // TMEM -> registers -> fused epilogue -> this warp's swizzled smem box
    // [32 rows][W cols] -> one TMA bulk store per slice (double-buffered): 4
    // shared-memory wavefronts per 512 B instead of 32 scattered global-store
    // wavefronts per warp instruction, and full-line writes into L2.  (Measured
    // time-neutral against direct 16-byte stores: these GEMMs are power-bound,
    // profiles/r01_epi_ab.md.)
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int half = (warp - 2) / 4;  // which half of the BN columns this warp drains
    constexpr int W = slice_width<EPI>();
    const uint32_t stg0 = base + L::kStgOffset + static_cast<uint32_t>(warp - 2) * L::kStgBytesPerWarp;
    int sbuf = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    const bool hint_c = l2hint & 8;  // output stores evict_first: C is not re-read by this GEMM
    const uint64_t pol_c = ptx::policy_evict_first();
    // Chunk signalling, deferred by one tile: tile i is counted when tile i+1's
    // accumulator is ready (its TMA stores have had a whole main loop to
    // complete, so the wait below is free) or at the end.  Counting right after
    // the stores stalled all 8 epilogue warps on the store round trip and the
    // fences every tile: +60% on the K = 1280 Out GEMM of cfg 4 (4,2).
    int pend_chunk = -1, pend_pj = 0;
    auto flush_signal = [&]() {
      if (pend_chunk < 0) return;
      if (lane == 0) {
        ptx::bulk_wait0();  // this warp's stores of the pending tile are complete ...
        asm volatile("fence.proxy.async.global;" ::: "memory");  // ... and ordered before generic accesses
      }
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
      // one release at system scope, cumulative over every epilogue warp's
      // stores through the barrier (NCCL, the stream-wait engine or a peer
      // rank reads them); a full fence.sc.sys per warp and tile stalled the
      // epilogue for microseconds on the short-K GEMMs
      if (warp == 2 && lane == 0) {
        uint32_t* ctr = push.p > 0 ? push.sig[pend_pj] + pend_chunk : sig + pend_chunk;
        asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
      }
      pend_chunk = -1;
    };
    for (int tile = unit; tile < num_tiles; tile += n_units) {
      int mt, nt, chunk;
      tile_coords(tile, mt_chunk, num_n, group_m, mt, nt, chunk);
      mt += m_lo;
      const int m0 = mt * BM * CG + BM * static_cast<int>(cta_rank);
      const int n0 = nt * BN;
      ptx::mbar_wait(tfull_bar(acc), acc_phase);
      ptx::tc_fence_after();
      if (sig != nullptr) flush_signal();  // the previous tile
      const int row = m0 + 32 * q + static_cast<int>(lane);
      // fused reduce-scatter: this CTA's 128 rows go to the owner of their row
      // slice (member pj), into its receive slot for this rank at row prow
      int pj = 0, prow = m0;
      if (push.p > 0) {
        const int rin = m0 - chunk * sig_rows;
        pj = rin / push.slice_rows;
        prow = chunk * push.slice_rows + (rin - pj * push.slice_rows);
      }
      const CUtensorMap* tm_out = push.p > 0 ? &push.tm[pj] : &tmC;
      const uint32_t tbase = tmem_base + (static_cast<uint32_t>(32 * q) << 16) + acc * BN;
      const int c_begin = half * (BN / 2 / W), c_end = (half + 1) * (BN / 2 / W);
      // software pipeline: the TMEM slice and side inputs of slice c+1 are in
      // flight while slice c is converted and staged
      uint32_t v[W];
      Side<W> sd;
      ptx::tmem_ld_slice<W>(tbase + W * c_begin, v);
      load_side<EPI, W>(sd, row, n0 + W * c_begin, M, N, ep);
#pragma unroll 1
      for (int c = c_begin; c < c_end; ++c) {
        ptx::tmem_wait_ld();
        float f[W];
#pragma unroll
        for (int j = 0; j < W; ++j) f[j] = __uint_as_float(v[j]);
        const Side<W> cur = sd;
        if (c + 1 < c_end) {
          ptx::tmem_ld_slice<W>(tbase + W * (c + 1), v);
          load_side<EPI, W>(sd, row, n0 + W * (c + 1), M, N, ep);
        }
        const int col0 = n0 + W * c;
        if (col0 >= N || m0 + 32 * q >= M) continue;  // warp-uniform: box entirely outside C
        const uint32_t stg = stg0 + static_cast<uint32_t>(sbuf) * 2048u;
        if (lane == 0) ptx::bulk_wait_read1();  // the store that last read this buffer is done reading
        __syncwarp();
        epilogue_chunk<EPI, W>(f, cur, static_cast<int>(lane), ep, stg);
        ptx::fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          if (hint_c) {
            ptx::tma_store_2d_hint(tm_out, stg, col0, prow + 32 * q, pol_c);
            if constexpr (EPI == EPI_BIAS_GELU)
              ptx::tma_store_2d_hint(&tmC2, stg + 32 * slice_row_bytes<EPI>(), col0, m0 + 32 * q, pol_c);
          } else {
            ptx::tma_store_2d(tm_out, stg, col0, prow + 32 * q);
            if constexpr (EPI == EPI_BIAS_GELU)
              ptx::tma_store_2d(&tmC2, stg + 32 * slice_row_bytes<EPI>(), col0, m0 + 32 * q);
          }
          ptx::bulk_commit();
        }
        sbuf ^= 1;
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2) {
          ptx::mbar_arrive_cluster(ptx::mapa_shared(tempty_bar(acc), 0));
        } else {
          ptx::mbar_arrive(tempty_bar(acc));
        }
      }
      if (sig != nullptr) {
        // counted once every epilogue warp's bulk stores of this tile are
        // complete and visible (system scope: NCCL / peer ranks read them)
        pend_chunk = chunk;
        pend_pj = pj;
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (sig != nullptr) flush_signal();  // the last tile
    if (lane == 0) ptx::bulk_wait0();  // staging smem stays valid until the last stores completed
  }

  ptx::tc_fence_before();
  if constexpr (CG == 2) {
    ptx::cluster_sync();
  } else {
    __syncthreads();
  }
  if (warp == 1) {
    ptx::tc_fence_after();
    if constexpr (CG == 2) {
      ptx::tmem_dealloc_cg2(tmem_base, TMEM_COLS);
    } else {
      ptx::tmem_dealloc(tmem_base, TMEM_COLS);
    }
  }
}

// ---------------------------------------------------------------- SM -> die map
// B200 is two dies; each address is homed in one die's L2 (2 KB granularity)
// and an SM reaches its own die's L2 ~30 cycles faster than the other's.  One
// CTA per SM times dependent L2 (.cg) loads to 256 addresses 2 KB apart; SMs
// of one die share the near/far pattern (profiles/r02_die_probe.md).
constexpr int kDieAddrs = 256, kDieStride = 2048, kDieReps = 8;

__global__ void die_latency_kernel(const uint32_t* buf, uint32_t* lat, int* smid_out) {
  extern __shared__ uint8_t pad[];
  if (threadIdx.x != 0) return;
  uint32_t smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  smid_out[blockIdx.x] = static_cast<int>(smid);
  pad[0] = 0;
  uint32_t dep = 0;
  for (int i = 0; i < kDieAddrs; ++i) {
    const uint32_t* p = buf + (static_cast<size_t>(i) * kDieStride) / 4;
    uint32_t idx = dep;  // the buffer holds zeros: every load's address depends on the previous value
    long long t0, t1;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0)::"memory");
#pragma unroll 1
    for (int r = 0; r < kDieReps; ++r) asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(idx) : "l"(p + idx) : "memory");
    asm volatile("add.u32 %0, %0, %1;" : "+r"(dep) : "r"(idx) : "memory");
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1)::"memory");
    lat[blockIdx.x * kDieAddrs + i] = static_cast<uint32_t>((t1 - t0) / kDieReps);
  }
  if (dep == 0xdeadbeefu) smid_out[blockIdx.x] = -1;  // keeps the load chain live
}

// Which SMs the CTA pairs of a 2-CTA cluster occupy (one CTA per SM).
__global__ void die_pair_kernel(int* out) {
  extern __shared__ uint8_t pad[];
  if (threadIdx.x != 0) return;
  uint32_t smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  pad[0] = 0;
  out[blockIdx.x] = static_cast<int>(smid);
}

std::atomic<bool> g_die_ready{false};
bool die_table_ready() { return g_die_ready.load(); }

struct DieTable {
  uint16_t* dev = nullptr;  // [num SMs]: die << 15 | pair index within the die
  int pairs[2] = {0, 0};
  bool ok = false;
};

// Measured once per process (ATP_DIE_AWARE=1 only).  Any inconsistency (not
// exactly two clusters of SMs, odd SM counts per die, a cluster pair spanning
// dies or changing between launches) disables the die-aware tile order.
const DieTable& die_table() {
  static DieTable t;
  static std::once_flag once;
  std::call_once(once, [] {
    const int nsm = num_sms();
    uint32_t *buf = nullptr, *lat = nullptr;
    int* ids = nullptr;
    const size_t bytes = static_cast<size_t>(kDieAddrs) * kDieStride;
    if (cudaMalloc(&buf, bytes) != cudaSuccess || cudaMalloc(&lat, sizeof(uint32_t) * nsm * kDieAddrs) != cudaSuccess ||
        cudaMalloc(&ids, sizeof(int) * 3 * nsm) != cudaSuccess)
      return;
    const int smem = 200 * 1024;  // one CTA per SM
    cudaMemset(buf, 0, bytes);
    cudaFuncSetAttribute(die_latency_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(die_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int it = 0; it < 2; ++it) die_latency_kernel<<<nsm, 32, smem>>>(buf, lat, ids);  // first pass warms L2
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nsm);
    cfg.blockDim = dim3(32);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, die_pair_kernel, ids + nsm);
    cudaLaunchKernelEx(&cfg, die_pair_kernel, ids + 2 * nsm);
    std::vector<uint32_t> h(static_cast<size_t>(nsm) * kDieAddrs);
    std::vector<int> hid(3 * nsm);
    bool good = cudaDeviceSynchronize() == cudaSuccess &&
                cudaMemcpy(h.data(), lat, h.size() * 4, cudaMemcpyDeviceToHost) == cudaSuccess &&
                cudaMemcpy(hid.data(), ids, hid.size() * 4, cudaMemcpyDeviceToHost) == cudaSuccess;
    cudaFree(buf);
    cudaFree(lat);
    cudaFree(ids);
    if (!good) {
      cudaGetLastError();
      return;
    }
    // correlate every SM's centred latency pattern with the lowest SM id's
    std::vector<double> z(h.size());
    for (int b = 0; b < nsm; ++b) {
      double mean = 0;
      for (int i = 0; i < kDieAddrs; ++i) mean += h[b * kDieAddrs + i];
      mean /= kDieAddrs;
      for (int i = 0; i < kDieAddrs; ++i) z[b * kDieAddrs + i] = h[b * kDieAddrs + i] - mean;
    }
    int ref = 0;
    for (int b = 1; b < nsm; ++b)
      if (hid[b] < hid[ref]) ref = b;
    std::vector<int> die_of_sm(nsm, -1);
    double nr = 0;
    for (int i = 0; i < kDieAddrs; ++i) nr += z[ref * kDieAddrs + i] * z[ref * kDieAddrs + i];
    for (int b = 0; b < nsm; ++b) {
      double dot = 0, nb = 0;
      for (int i = 0; i < kDieAddrs; ++i) {
        dot += z[b * kDieAddrs + i] * z[ref * kDieAddrs + i];
        nb += z[b * kDieAddrs + i] * z[b * kDieAddrs + i];
      }
      const double c = dot / std::sqrt(nr * nb + 1e-30);
      if (std::fabs(c) < 0.3) return;  // no clear two-die structure
      if (hid[b] < 0 || hid[b] >= nsm || die_of_sm[hid[b]] != -1) return;
      die_of_sm[hid[b]] = c > 0 ? 0 : 1;
    }
    // cluster pairs: both launches identical (as sets), each pair inside one die
    std::vector<int> partner(nsm, -1);
    for (int l = 1; l <= 2; ++l)
      for (int c = 0; c + 1 < nsm; c += 2) {
        const int a = hid[l * nsm + c], b = hid[l * nsm + c + 1];
        if (a < 0 || b < 0 || a >= nsm || b >= nsm || die_of_sm[a] != die_of_sm[b]) return;
        if (l == 1) {
          partner[a] = b;
          partner[b] = a;
        } else if (partner[a] != b) {
          return;
        }
      }
    std::vector<uint16_t> tab(nsm, 0);
    int pairs[2] = {0, 0};
    for (int sm = 0; sm < nsm; ++sm) {  // pair index = order of the pair's lower SM id within its die
      const int p = partner[sm];
      if (p < 0) return;
      if (sm < p) {
        const int d = die_of_sm[sm];
        tab[sm] = tab[p] = static_cast<uint16_t>((d << 15) | pairs[d]);
        ++pairs[d];
      }
    }
    if (pairs[0] == 0 || pairs[1] == 0) return;
    if (cudaMalloc(&t.dev, sizeof(uint16_t) * nsm) != cudaSuccess) return;
    cudaMemcpy(t.dev, tab.data(), sizeof(uint16_t) * nsm, cudaMemcpyHostToDevice);
    t.pairs[0] = pairs[0];
    t.pairs[1] = pairs[1];
    t.ok = true;
  });
  g_die_ready = true;
  return t;
}

// ATP_DIE_AWARE=1: die-aware tile order for the all-SM CTA-pair GEMMs (A/B runs).
bool die_aware() {
  static const bool on = [] {
    const char* e = getenv("ATP_DIE_AWARE");
    return e && e[0] == '1';
  }();
  return on;
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

bool get_encode() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode != nullptr;
}

// 2-D bf16 tensor map over a row-major [rows, cols] matrix with row pitch ld
// (elements); box = [box_rows, box_cols], 128B swizzle, OOB -> zero.
bool make_tmap(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
               int box_cols) {
  if (!get_encode()) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// L2 cache hints of the TMA loads / stores (ATP_L2HINT bitmask, A/B runs):
// 1 = A evict_last, 2 = B evict_first, 4 = B evict_last, 8 = C stores evict_first.
int l2hint() {
  static const int v = [] {
    const char* e = getenv("ATP_L2HINT");
    return e ? atoi(e) : 0;
  }();
  return v;
}

// Serpentine K order across persistent rounds (ATP_KSERP=0 disables; A/B runs).
int kserp() {
  static const int v = [] {
    const char* e = getenv("ATP_KSERP");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return v;
}

template <int CG, int BN, int STAGES, int EPI, bool A_MN, bool B_MN>
cudaError_t launch_t(const GemmDesc& d, int grid, cudaStream_t st) {
  using L = SmemLayout<CG, BN, STAGES>;
  auto kern = gemm_sm100_kernel<CG, BN, STAGES, EPI, A_MN, B_MN>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kBytes);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = L::kBytes;
  cfg.stream = st;
  static const bool pdl = [] {  // ATP_PDL=0 disables programmatic dependent launch (A/B runs)
    const char* e = getenv("ATP_PDL");
    return !(e && e[0] == '0');
  }();
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl && d.pdl && d.gate == nullptr) ? 2 : 1;
  // die-aware tile order: CTA pairs on every SM (one CTA per SM), no chunk
  // signalling / gating / push (their tile order is chunk-major), >= 4 M-tiles
  const uint16_t* die_tab = nullptr;
  int dp0 = 0, dp1 = 0;
  cudaStreamCaptureStatus capturing = cudaStreamCaptureStatusNone;
  if (CG == 2 && die_aware()) cudaStreamIsCapturing(st, &capturing);
  // (the table is measured outside any graph capture: the first uncaptured call sets it up)
  if (CG == 2 && die_aware() && grid == num_sms() && d.sig == nullptr && d.gate == nullptr && d.push.p == 0 &&
      (d.M + 255) / 256 >= 4 && (capturing == cudaStreamCaptureStatusNone || die_table_ready())) {
    const DieTable& t = die_table();
    if (t.ok && 2 * (t.pairs[0] + t.pairs[1]) == grid) {
      die_tab = t.dev;
      dp0 = t.pairs[0];
      dp1 = t.pairs[1];
    }
  }
  return cudaLaunchKernelEx(&cfg, kern, d.tmA, d.tmB, d.tmC, d.tmC2, d.M, d.N, d.K, d.ep, d.sig, d.sig_rows, d.gate,
                            d.gate_target, d.group_m > 0 ? d.group_m : 16, kserp(), l2hint(), d.push, die_tab, dp0,
                            dp1);
}

template <int CG, int BN, int STAGES, bool A_MN, bool B_MN>
cudaError_t launch_epi(const GemmDesc& d, int grid, cudaStream_t st) {
  switch (d.epi) {
    case EPI_BF16: return launch_t<CG, BN, STAGES, EPI_BF16, A_MN, B_MN>(d, grid, st);
    case EPI_F32: return launch_t<CG, BN, STAGES, EPI_F32, A_MN, B_MN>(d, grid, st);
    case EPI_RESID: return launch_t<CG, BN, STAGES, EPI_RESID, A_MN, B_MN>(d, grid, st);
    case EPI_BIAS_GELU: return launch_t<CG, BN, STAGES, EPI_BIAS_GELU, A_MN, B_MN>(d, grid, st);
    case EPI_DGELU: return launch_t<CG, BN, STAGES, EPI_DGELU, A_MN, B_MN>(d, grid, st);
  }
  return cudaErrorInvalidValue;
}

template <int CG, int BN, int STAGES>
cudaError_t launch_bn(const GemmDesc& d, int grid, cudaStream_t st) {
  if (!d.a_mn && d.b_mn) return launch_epi<CG, BN, STAGES, false, true>(d, grid, st);
  if (!d.a_mn && !d.b_mn) return launch_epi<CG, BN, STAGES, false, false>(d, grid, st);
  if (d.a_mn && d.b_mn) return launch_epi<CG, BN, STAGES, true, true>(d, grid, st);
  return cudaErrorInvalidValue;  // (MN, K) is not used by the layer
}

int g_num_sms = 0;

// ATP_GEMM_MODE=1 forces single-CTA tiles (A/B comparison of the two kernels).
int gemm_mode() {
  static int mode = [] {
    const char* e = getenv("ATP_GEMM_MODE");
    return e ? atoi(e) : 0;
  }();
  return mode;
}

}  // namespace

// M-tiles per raster group (tiles sweep all N-tiles of a group before the next
// group).  Default: when the whole B operand (N x K, bf16) fits ~72 MB of L2,
// 2 — every round sweeps all of B, which then stays L2-resident while A
// streams through once; otherwise 16 when one M-tile's A panel (rows x K) is
// <= ~2 MB (K <= 4096 at 256-row tiles), else 8: the ~74 tiles of a
// persistent round then cover a near-square block of panels, and with the
// serpentine K order consecutive rounds meet their shared panels in L2.
// Measured per-GEMM DRAM reads over g = 2..32
// (profiles/r01_groupm_dram_sweep.log): 8.97 GB per step predicted vs 9.80 GB
// for the earlier rule (largest g whose panel group fits ~40 MB of L2) and
// 9.57 GB for a fixed 16.  ATP_GROUP_M=g > 0 fixes it.
int raster_group_m(int rows_per_mtile, int N, int K) {
  static const int env = [] {
    const char* e = getenv("ATP_GROUP_M");
    return e ? atoi(e) : -1;
  }();
  if (env > 0) return env;
  if (static_cast<double>(N) * K * 2.0 <= 72e6) return 2;
  const double panel = static_cast<double>(rows_per_mtile) * K * 2.0;
  return panel <= 2.2e6 ? 16 : 8;
}

// Output map of the epilogue's TMA stores: [rows, cols] (pitch ld elements of
// esz bytes), box [32 rows][box_cols], swizzle = the box row's bytes (32 / 64).
bool make_tmap_out(CUtensorMap* m, const void* ptr, int esz, int64_t rows, int64_t cols, int64_t ld, int box_cols) {
  if (!get_encode()) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * esz)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), 32u};
  cuuint32_t estr[2] = {1, 1};
  const int rb = box_cols * esz;
  return g_encode(m, esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  rb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool tmap_bf16_2d(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                  int box_cols) {
  return make_tmap(m, ptr, rows, cols, ld, box_rows, box_cols);
}

bool tmap_f32_2d(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                 int box_cols) {
  if (!get_encode()) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 4)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  return g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

// N tile 256 when N is a multiple of 256 or large, else 128; CTA pairs for big
// tiles (M >= 256 and a 256-wide N tile), single CTAs otherwise.
void gemm_plan_tile(int M, int N, int* bn, int* cg) {
  *bn = (N % 256 == 0 || N > 1024) ? 256 : 128;
  *cg = (*bn == 256 && M >= 256 && gemm_mode() != 1) ? 2 : 1;
}

int gemm_tiles(const GemmDesc& d) {
  return ((d.M + BM * d.cg - 1) / (BM * d.cg)) * ((d.N + d.bn - 1) / d.bn);
}

// Validate and build the TMA descriptors of one GEMM.  Returns a message on error.
const char* gemm_prepare(GemmDesc& d, const void* A, int64_t lda, bool a_mn, const void* B, int64_t ldb,
                         bool b_mn, int M, int N, int K) {
  if (M <= 0 || N <= 0 || K <= 0) return "gemm: M, N, K must be positive";
  if (a_mn && !b_mn) return "gemm: operand arrangement (MN, K) unsupported";
  if ((N % 8) != 0 || (K % 8) != 0 || (a_mn && (M % 8) != 0)) return "gemm: N, K (and M for MN-major A) must be multiples of 8";
  if ((lda % 8) != 0 || (ldb % 8) != 0) return "gemm: leading dimensions must be multiples of 8 elements";
  if ((reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15)) return "gemm: operands must be 16-byte aligned";
  d.M = M;
  d.N = N;
  d.K = K;
  d.a_mn = a_mn;
  d.b_mn = b_mn;
  if (d.bn != 128 && d.bn != 256) gemm_plan_tile(M, N, &d.bn, &d.cg);
  if (d.cg != 1 && d.cg != 2) d.cg = (d.bn == 256 && M >= 256 && gemm_mode() != 1) ? 2 : 1;
  if (d.cg == 2 && d.bn != 256) d.cg = 1;
  d.group_m = raster_group_m(d.cg == 2 ? 256 : BM, N, K);  // after cg is final (rows per M-tile)
  bool ok;
  if (!a_mn)
    ok = make_tmap(&d.tmA, A, M, K, lda, BM, BK);
  else
    ok = make_tmap(&d.tmA, A, K, M, lda, BK, 64);
  if (!ok) return "gemm: cuTensorMapEncodeTiled failed for A";
  if (!b_mn)
    ok = make_tmap(&d.tmB, B, N, K, ldb, d.bn / d.cg, BK);
  else
    ok = make_tmap(&d.tmB, B, K, N, ldb, BK, 64);
  if (!ok) return "gemm: cuTensorMapEncodeTiled failed for B";
  // epilogue output maps (the EpiParams must be final here)
  const int epi = d.epi;
  const int esz = epi == EPI_F32 ? 4 : 2;
  const int w = epi == EPI_BF16 ? 32 : 16;  // slice_width<EPI>()
  if (d.ep.C == nullptr || (reinterpret_cast<uintptr_t>(d.ep.C) & 15) || (d.ep.ldc * esz) % 16)
    return "gemm: output must be 16-byte aligned with a 16-byte multiple row pitch";
  if (!make_tmap_out(&d.tmC, d.ep.C, esz, M, N, d.ep.ldc, w)) return "gemm: cuTensorMapEncodeTiled failed for C";
  d.tmC2 = d.tmC;
  if (epi == EPI_BIAS_GELU) {
    if (d.ep.C2 == nullptr || (reinterpret_cast<uintptr_t>(d.ep.C2) & 15) || (d.ep.ldc2 * 2) % 16)
      return "gemm: GeLU output must be 16-byte aligned with a 16-byte multiple row pitch";
    if (!make_tmap_out(&d.tmC2, d.ep.C2, 2, M, N, d.ep.ldc2, w)) return "gemm: cuTensorMapEncodeTiled failed for C2";
  }
  return nullptr;
}

cudaError_t gemm_launch(const GemmDesc& d, cudaStream_t st) {
  if (d.dtype == 1) return gemm_launch_f32(d, st);
  int sms = d.max_ctas > 0 ? d.max_ctas : num_sms();
  const int units = sms / d.cg > 0 ? sms / d.cg : 1;
  const int tiles = gemm_tiles(d);
  const int grid = (tiles < units ? tiles : units) * d.cg;
  if (d.cg == 2) return launch_bn<2, 256, 6>(d, grid, st);
  if (d.bn == 256) return launch_bn<1, 256, 4>(d, grid, st);
  return launch_bn<1, 128, 6>(d, grid, st);
}

}  // namespace atp
