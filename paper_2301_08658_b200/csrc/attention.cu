// Attention core: O = softmax(Q K^T / sqrt(d)) V per
// sequence and head (Eq. 1), causal (reading G30), head dim 128,
// on tcgen05 tensor cores with TMEM accumulators.
//
// Input: one rank's head block of the QKV activations, token-major
// [T, 3 * heads * 128] with head-interleaved columns (head j: q at 3j*128,
// k at 3j*128 + 128, v at 3j*128 + 256; reading G19).  Rows are whole
// sequences of `seq` tokens (seq % 128 == 0).
//
// Forward: one CTA per (128-query block, head, sequence), heaviest causal
// blocks first.  Warp roles:
//   warp 0     TMA: Q once, then K_j / V_j double-buffered (one tensor map over
//              the QKV block, 64 x 128 boxes, 128B swizzle)
//   warp 1     MMA issuer: S_{j+1} = Q K_{j+1}^T into the other TMEM S buffer
//              while the softmax works on S_j, then O += P_j V_j (V as an
//              MN-major B operand, P from shared memory)
//   warps 4-7  softmax, one thread per query row (TMEM lane = row): online
//              softmax in the log2 domain with LAZY rescaling — O (in TMEM)
//              is corrected only when the running row max grows by more than
//              8 (a factor 256), so p = exp2(s - m) stays <= 256 and the
//              correction pass is rare; P (bf16) goes to shared memory in the
//              SW128 K-major layout the MMA reads.
// TMEM: S0 [0,128) S1 [128,256) O [256,384) of a 512-column allocation.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstdint>

#include "atp_internal.h"
#include "attention.h"
#include "sm100_ptx.cuh"

namespace atp {

namespace {

constexpr int HD = 128;                  // head dim
constexpr int BQ = 128;                  // query rows per CTA
constexpr int BKV = 128;                 // keys per block
constexpr uint32_t kHalf = 128 * 128;    // one 64-column SW128 box of 128 rows (bytes)
constexpr uint32_t kTile = 2 * kHalf;    // [128 rows][128 cols] bf16
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// 2^x (MUFU.EX2, flush-to-zero; 2^-inf = 0)
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Blackwell paired fp32 ops (FFMA2 / FADD2: two lanes of fp32 per instruction)
// and the three-input max (FMNMX3), to halve the softmax's FMA/ALU issue.
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2unpack(uint64_t r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// Byte offset of the 16-byte chunk `c16` (8 bf16 columns) of row r in a
// [128 rows][128 cols] tile stored as two SW128 boxes of 64 columns.
__device__ __forceinline__ uint32_t sw128_off(int r, int c16) {
  return static_cast<uint32_t>((c16 >> 3) * kHalf + r * 128 + (((c16 & 7) ^ (r & 7)) << 4));
}

// K-major operand descriptor for K-step kk (16 columns) of a 128x128 tile.
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t tile, int kk) {
  return ptx::smem_desc_sw128(tile + (kk >> 2) * kHalf + (kk & 3) * 32, 16, 1024);
}
// MN-major operand descriptor (MN = the 128 tile columns, K = the 128 tile rows).
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t tile, int kk) {
  return ptx::smem_desc_sw128(tile + kk * 2048, kHalf, 1024);
}

struct FwdParams {
  int T, seq, heads, causal;
  int grouped;  // CTA order: G > 0 = chunks of G (sequence, head) groups, heaviest first inside a chunk (L2 reuse)
  float scale_log2;  // log2(e) / sqrt(d)
  __nv_bfloat16* ctx;
  int64_t ld_ctx;
  float* lse;  // [heads][T], natural log
  // split-KV (forward v2 on grids smaller than the GPU): kv_split CTAs per
  // query-tile pair, each over a contiguous share of its KV blocks, writing
  // unnormalised O (fp32) and (max, sum) per row to opart / mlpart; a combine
  // kernel merges them.  kv_split == 1: the CTA normalises and writes ctx, lse.
  int kv_split = 1;
  float* opart = nullptr;   // [kv_split][T][heads * 128]
  float* mlpart = nullptr;  // [kv_split][T][heads][2]: running max (log2 domain, scaled), row sum
};

// CTA order.  G == 0: heaviest work first across the whole grid.  G > 0: the
// (sequence, head) groups are taken G at a time (a chunk of ~2 waves of CTAs
// whose K/V or Q/dO stay in L2 while every block of the chunk re-reads them),
// heaviest first inside a chunk (so the tail stays light).  `per_group` =
// CTAs of one group, `j` = heaviness rank inside the group (0 = heaviest).
__device__ __forceinline__ void cta_order(int G, int n_groups, int per_group, int& j, int& group,
                                          int b = static_cast<int>(blockIdx.x)) {
  if (G <= 0) {
    j = b / n_groups;
    group = b % n_groups;
    return;
  }
  const int c = b / (G * per_group);
  const int first = c * G;
  const int gc = min(G, n_groups - first);
  const int in = b - first * per_group;
  j = in / gc;
  group = first + in % gc;
}

// Block index -> (query block, head, sequence); causal: heaviest query blocks first.
__device__ __forceinline__ void fwd_coords(const FwdParams& p, int& qb, int& head, int& sq) {
  const int nqb = p.seq / BQ, nseq = p.T / p.seq;
  const int per = p.heads * nseq;
  qb = static_cast<int>(blockIdx.x) / per;
  if (p.causal) qb = nqb - 1 - qb;
  const int rest = static_cast<int>(blockIdx.x) % per;
  head = rest % p.heads;
  sq = rest / p.heads;
}

__global__ void __launch_bounds__(256, 1) attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_qkv, FwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t sQ = base, sP = base + 5 * kTile;
  auto sK = [&](int s) { return base + kTile + s * 2 * kTile; };
  auto sV = [&](int s) { return base + 2 * kTile + s * 2 * kTile; };
  const uint32_t bars = base + 6 * kTile;
  const uint32_t q_full = bars, p_full = bars + 8, o_done = bars + 16;
  auto kv_full = [&](int s) { return bars + 24 + 8 * s; };
  auto kv_empty = [&](int s) { return bars + 40 + 8 * s; };
  auto s_full = [&](int s) { return bars + 56 + 8 * s; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw + (bars + 72 - raw));

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  int qb, head, sq;
  fwd_coords(p, qb, head, sq);
  const int row0 = sq * p.seq, qrow = row0 + qb * BQ;
  const int nkv = p.causal ? qb + 1 : p.seq / BKV;
  const int qcol = head * 3 * HD;

  if (threadIdx.x == 0) {
    ptx::mbar_init(q_full, 1);
    ptx::mbar_init(p_full, 128);
    ptx::mbar_init(o_done, 1);
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(kv_full(s), 1);
      ptx::mbar_init(kv_empty(s), 1);
      ptx::mbar_init(s_full(s), 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) {
    ptx::tmem_alloc(ptx::smem_u32(tmem_slot), 512);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer
      ptx::prefetch_tmap(&tm_qkv);
      ptx::mbar_arrive_expect_tx(q_full, kTile);
      ptx::tma_load_2d(sQ, &tm_qkv, q_full, qcol, qrow);
      ptx::tma_load_2d(sQ + kHalf, &tm_qkv, q_full, qcol + 64, qrow);
      for (int j = 0; j < nkv; ++j) {
        const int s = j & 1;
        ptx::mbar_wait(kv_empty(s), ((j >> 1) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(kv_full(s), 2 * kTile);
        const int kr = row0 + j * BKV;
        ptx::tma_load_2d(sK(s), &tm_qkv, kv_full(s), qcol + HD, kr);
        ptx::tma_load_2d(sK(s) + kHalf, &tm_qkv, kv_full(s), qcol + HD + 64, kr);
        ptx::tma_load_2d(sV(s), &tm_qkv, kv_full(s), qcol + 2 * HD, kr);
        ptx::tma_load_2d(sV(s) + kHalf, &tm_qkv, kv_full(s), qcol + 2 * HD + 64, kr);
      }
      for (int j = nkv; j < nkv + 2; ++j) ptx::mbar_wait(kv_empty(j & 1), ((j >> 1) & 1) ^ 1);  // tail
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------ MMA issuer
      constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(128, 128, 0, 0);
      constexpr uint32_t idesc_o = ptx::idesc_bf16_f32(128, 128, 0, 1);
      ptx::mbar_wait(q_full, 0);
      auto issue_s = [&](int j) {
        const int s = j & 1;
        ptx::mbar_wait(kv_full(s), (j >> 1) & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          ptx::mma_bf16_ss(tmem + s * 128, desc_kmajor(sQ, kk), desc_kmajor(sK(s), kk), idesc_s, kk > 0 ? 1u : 0u);
        ptx::mma_commit(s_full(s));
      };
      issue_s(0);
      for (int j = 0; j < nkv; ++j) {
        if (j + 1 < nkv) issue_s(j + 1);  // its S buffer was released with P_{j-1}
        ptx::mbar_wait(p_full, j & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk)
          ptx::mma_bf16_ss(tmem + 256, desc_kmajor(sP, kk), desc_mnmajor(sV(j & 1), kk), idesc_o,
                           (j | kk) != 0 ? 1u : 0u);
        ptx::mma_commit(o_done);
        ptx::mma_commit(kv_empty(j & 1));
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ softmax (row r of the query block)
    const int q4 = warp - 4;
    const int r = q4 * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    float m_run = -INFINITY, l = 0.f;
    for (int j = 0; j < nkv; ++j) {
      const int s = j & 1;
      ptx::mbar_wait(s_full(s), (j >> 1) & 1);
      ptx::tc_fence_after();
      float sv[BKV];
#pragma unroll
      for (int c = 0; c < BKV / 32; ++c) {
        uint32_t u[32];
        ptx::tmem_ld_32x32b_x32(tmem + lane_off + s * 128 + c * 32, u);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) sv[c * 32 + i] = __uint_as_float(u[i]) * p.scale_log2;
      }
      if (p.causal && j == qb) {
#pragma unroll
        for (int c = 0; c < BKV; ++c)
          if (c > r) sv[c] = -INFINITY;
      }
      float mb = sv[0];
#pragma unroll
      for (int c = 1; c < BKV; ++c) mb = fmaxf(mb, sv[c]);
      const bool need = mb > m_run + 8.f;
      if (j > 0) {
        ptx::mbar_wait(o_done, (j - 1) & 1);  // PV_{j-1} done: O stable, P buffer free
        ptx::tc_fence_after();
      }
      if (__any_sync(0xffffffffu, need)) {  // warp-uniform: tcgen05.ld/st are warp-collective
        const float m_new = fmaxf(m_run, mb);
        const float f = exp2f(m_run - m_new);
        l *= f;
        if (j > 0) {
#pragma unroll
          for (int c = 0; c < HD / 32; ++c) {
            uint32_t u[32];
            const uint32_t ta = tmem + lane_off + 256 + c * 32;
            ptx::tmem_ld_32x32b_x32(ta, u);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(__uint_as_float(u[i]) * f);
            ptx::tmem_st_32x32b_x32(ta, u);
          }
          ptx::tmem_wait_st();
        }
        m_run = m_new;
      }
      float rs = 0.f;
#pragma unroll
      for (int c16 = 0; c16 < BKV / 8; ++c16) {
        float e[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          e[i] = exp2f(sv[c16 * 8 + i] - m_run);
          rs += e[i];
        }
        st_shared_v4(sP + sw128_off(r, c16), pack_bf16(e[0], e[1]), pack_bf16(e[2], e[3]), pack_bf16(e[4], e[5]),
                     pack_bf16(e[6], e[7]));
      }
      l += rs;
      ptx::fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor core
      ptx::tc_fence_before();
      ptx::mbar_arrive(p_full);
    }
    // ---- epilogue: O / l -> ctx (bf16), log-sum-exp -> lse
    ptx::mbar_wait(o_done, (nkv - 1) & 1);
    ptx::tc_fence_after();
    const float inv = 1.f / l;
    __nv_bfloat16* orow = p.ctx + static_cast<int64_t>(qrow + r) * p.ld_ctx + head * HD;
#pragma unroll
    for (int c = 0; c < HD / 32; ++c) {
      uint32_t u[32];
      ptx::tmem_ld_32x32b_x32(tmem + lane_off + 256 + c * 32, u);
      ptx::tmem_wait_ld();
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        uint4 w;
        w.x = pack_bf16(__uint_as_float(u[8 * v + 0]) * inv, __uint_as_float(u[8 * v + 1]) * inv);
        w.y = pack_bf16(__uint_as_float(u[8 * v + 2]) * inv, __uint_as_float(u[8 * v + 3]) * inv);
        w.z = pack_bf16(__uint_as_float(u[8 * v + 4]) * inv, __uint_as_float(u[8 * v + 5]) * inv);
        w.w = pack_bf16(__uint_as_float(u[8 * v + 6]) * inv, __uint_as_float(u[8 * v + 7]) * inv);
        *reinterpret_cast<uint4*>(orow + c * 32 + 8 * v) = w;
      }
    }
    p.lse[static_cast<int64_t>(head) * p.T + qrow + r] = (m_run + log2f(l)) * kLn2;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

constexpr int kFwdSmem = 6 * kTile + 128 + 1024;

// ---------------------------------------------------------------- forward v2
// Two 128-row query tiles per CTA (query blocks 2m and 2m+1 of a sequence)
// share each K/V block; each tile has its own softmax warpgroup (warps 2-5:
// tile 0, warps 6-9: tile 1).  P goes back into TMEM over its S columns
// (bf16 pairs) and is the A operand of O += P V straight from TMEM, so the
// MMA warp ping-pongs: PV_0(j), S_0(j+1), PV_1(j), S_1(j+1) — the tensor core
// works on one tile while the other tile's softmax runs.  The score row is
// read from TMEM twice (max pass, then exp pass) in 32-column slices to keep
// register pressure low.  TMEM: tile t at [256t, 256t+256): S/P [0,128),
// O [128,256).  Shared memory: Q0, Q1, and two K/V stages (192 KB).
__global__ void __launch_bounds__(320, 1) attn_fwd2_kernel(const __grid_constant__ CUtensorMap tm_qkv, FwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  auto sQ = [&](int t) { return base + t * kTile; };
  auto sK = [&](int s) { return base + 2 * kTile + s * 2 * kTile; };
  auto sV = [&](int s) { return base + 3 * kTile + s * 2 * kTile; };
  const uint32_t bars = base + 6 * kTile;
  const uint32_t q_full = bars;
  auto kv_full = [&](int s) { return bars + 8 + 8 * s; };
  auto kv_empty = [&](int s) { return bars + 24 + 8 * s; };
  auto s_full = [&](int t) { return bars + 40 + 8 * t; };
  auto p_full = [&](int t) { return bars + 56 + 8 * t; };
  auto o_done = [&](int t) { return bars + 72 + 8 * t; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw + (bars + 88 - raw));

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nq = p.seq / BQ, nm = (nq + 1) / 2, nseq = p.T / p.seq;
  const int per = p.heads * nseq;
  int m, rest;
  const int split = static_cast<int>(blockIdx.x) % p.kv_split;
  cta_order(p.grouped, per, nm, m, rest, static_cast<int>(blockIdx.x) / p.kv_split);
  if (p.causal) m = nm - 1 - m;  // heaviest first
  const int head = rest % p.heads, sq = rest / p.heads;
  const int row0 = sq * p.seq;
  int qblk[2], n[2];
  for (int t = 0; t < 2; ++t) {
    qblk[t] = 2 * m + t;
    n[t] = qblk[t] < nq ? (p.causal ? qblk[t] + 1 : nq) : 0;
  }
  const int nkv_all = n[0] > n[1] ? n[0] : n[1];
  // this CTA's KV blocks [j0, j1); tile t runs [j0, min(j1, n[t])) -- nl[t] steps
  const int kv_per = (nkv_all + p.kv_split - 1) / p.kv_split;
  const int j0 = min(nkv_all, split * kv_per), j1 = min(nkv_all, j0 + kv_per);
  const int nkv = j1 - j0;
  int nl[2];
  for (int t = 0; t < 2; ++t) nl[t] = max(0, min(j1, n[t]) - j0);
  const int qcol = head * 3 * HD;

  if (threadIdx.x == 0) {
    ptx::mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(kv_full(s), 1);
      ptx::mbar_init(kv_empty(s), 1);
      ptx::mbar_init(s_full(s), 1);
      ptx::mbar_init(p_full(s), 128);
      ptx::mbar_init(o_done(s), 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc(ptx::smem_u32(tmem_slot), 512);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);

  if (warp == 0) {
    if (lane == 0) {
      ptx::prefetch_tmap(&tm_qkv);
      ptx::mbar_arrive_expect_tx(q_full, ((nl[0] > 0 ? 1 : 0) + (nl[1] > 0 ? 1 : 0)) * kTile);
      for (int t = 0; t < 2; ++t) {
        if (nl[t] == 0) continue;
        const int qr = row0 + qblk[t] * BQ;
        ptx::tma_load_2d(sQ(t), &tm_qkv, q_full, qcol, qr);
        ptx::tma_load_2d(sQ(t) + kHalf, &tm_qkv, q_full, qcol + 64, qr);
      }
      for (int j = 0; j < nkv; ++j) {  // local step j = KV block j0 + j
        const int s = j & 1;
        ptx::mbar_wait(kv_empty(s), ((j >> 1) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(kv_full(s), 2 * kTile);
        const int kr = row0 + (j0 + j) * BKV;
        ptx::tma_load_2d(sK(s), &tm_qkv, kv_full(s), qcol + HD, kr);
        ptx::tma_load_2d(sK(s) + kHalf, &tm_qkv, kv_full(s), qcol + HD + 64, kr);
        ptx::tma_load_2d(sV(s), &tm_qkv, kv_full(s), qcol + 2 * HD, kr);
        ptx::tma_load_2d(sV(s) + kHalf, &tm_qkv, kv_full(s), qcol + 2 * HD + 64, kr);
      }
    }
  } else if (warp == 1) {
    {  // the whole warp runs the issue loop; each tcgen05 op is issued by one elected lane
      constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(128, 128, 0, 0);
      constexpr uint32_t idesc_o = ptx::idesc_bf16_f32(128, 128, 0, 1);
      auto adv = [](uint64_t d, uint32_t bytes) { return d + (bytes >> 4); };
      const uint64_t q_kmaj[2] = {ptx::smem_desc_sw128(sQ(0), 16, 1024), ptx::smem_desc_sw128(sQ(1), 16, 1024)};
      const uint64_t k_kmaj[2] = {ptx::smem_desc_sw128(sK(0), 16, 1024), ptx::smem_desc_sw128(sK(1), 16, 1024)};
      const uint64_t v_mnmaj[2] = {ptx::smem_desc_sw128(sV(0), kHalf, 1024), ptx::smem_desc_sw128(sV(1), kHalf, 1024)};
      int kv_seen = -1;
      auto need_kv = [&](int j) {
        if (j > kv_seen) {
          ptx::mbar_wait(kv_full(j & 1), (j >> 1) & 1);
          ptx::tc_fence_after();
          kv_seen = j;
        }
      };
      auto issue_s = [&](int t, int j) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          ptx::mma_bf16_ss_w(tmem + 256 * t, adv(q_kmaj[t], (kk >> 2) * kHalf + (kk & 3) * 32),
                             adv(k_kmaj[j & 1], (kk >> 2) * kHalf + (kk & 3) * 32), idesc_s, kk > 0 ? 1u : 0u);
        ptx::mma_commit_w(s_full(t));
      };
      if (nkv > 0) {
        ptx::mbar_wait(q_full, 0);
        need_kv(0);
      }
      for (int t = 0; t < 2; ++t)
        if (nl[t] > 0) issue_s(t, 0);
      for (int j = 0; j < nkv; ++j) {  // local steps; tile t is active for j < nl[t]
        for (int t = 0; t < 2; ++t) {
          if (j >= nl[t]) continue;
          ptx::mbar_wait(p_full(t), j & 1);
          ptx::tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk)
            ptx::mma_bf16_ts_w(tmem + 256 * t + 128, tmem + 256 * t + kk * 8, adv(v_mnmaj[j & 1], kk * 2048), idesc_o,
                               (j | kk) != 0 ? 1u : 0u);
          if (j + 1 == nl[t]) ptx::mma_commit_w(o_done(t));  // one phase: the final O (nobody waits on the others)
          if (j + 1 < nl[t]) {
            need_kv(j + 1);
            issue_s(t, j + 1);
          }
        }
        ptx::mma_commit_w(kv_empty(j & 1));
      }
    }
  } else {
    // ------------------------------------------------ softmax of tile t, row r
    const int t = (warp - 2) / 4;
    const int nt = t ? nl[1] : nl[0], qbt = t ? qblk[1] : qblk[0];
    const int q4 = warp % 4;  // TMEM lane quarter this warp may access
    const int r = q4 * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const uint32_t tS = tmem + lane_off + 256 * t, tO = tS + 128;
    float m_run = -INFINITY, l = 0.f;
    for (int j = 0; j < nt; ++j) {
      ptx::mbar_wait(s_full(t), j & 1);
      ptx::tc_fence_after();
      uint32_t u[BKV / 32][32];  // the whole score row: four loads, one wait
#pragma unroll
      for (int c = 0; c < BKV / 32; ++c) ptx::tmem_ld_32x32b_x32(tS + c * 32, u[c]);
      ptx::tmem_wait_ld();
      if (p.causal && j0 + j == qbt) {  // diagonal block: keys after the query row are masked
#pragma unroll
        for (int c = 0; c < BKV; ++c)
          if (c > r) u[c / 32][c % 32] = __float_as_uint(-INFINITY);
      }
      // row max as an 8-way tree (a 128-long dependent fmax chain was ~500 cycles)
      float mx[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mx[i] = __uint_as_float(u[i / 32][i % 32]);
#pragma unroll
      for (int c = 8; c < BKV; c += 2)
        mx[(c / 2) % 8] = fmax3(mx[(c / 2) % 8], __uint_as_float(u[c / 32][c % 32]), __uint_as_float(u[c / 32][c % 32 + 1]));
      float mb = fmaxf(fmax3(mx[0], mx[1], mx[2]), fmax3(fmax3(mx[3], mx[4], mx[5]), mx[6], mx[7]));
      mb *= p.scale_log2;
      // Lazy rescale (warp-uniform: tcgen05.ld/st are warp-collective).  P is
      // written with the new max first; O is corrected afterwards, once the
      // score row is dead, still before p_full releases PV(j).  PV(j-1) is
      // complete here: S(j) was issued after it.
      const bool rescale = __any_sync(0xffffffffu, mb > m_run + 8.f);
      float f = 1.f;
      if (rescale) {
        const float m_new = fmaxf(m_run, mb);
        f = ex2(m_run - m_new);
        m_run = m_new;
      }
      // x = s * scale - m and the row sums on pairs of columns (FFMA2 / FADD2)
      const uint64_t sc2 = f2pack(p.scale_log2, p.scale_log2), nm2 = f2pack(-m_run, -m_run);
      uint64_t rsv[2] = {f2pack(0.f, 0.f), f2pack(0.f, 0.f)};  // 2 x 2 partial row sums
#pragma unroll
      for (int c = 0; c < BKV / 32; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float x0, x1;
          f2unpack(ffma2(f2pack(__uint_as_float(u[c][2 * i]), __uint_as_float(u[c][2 * i + 1])), sc2, nm2), x0, x1);
          const float e0 = ex2(x0), e1 = ex2(x1);
          rsv[i % 2] = fadd2(rsv[i % 2], f2pack(e0, e1));
          pk[i] = pack_bf16(e0, e1);
        }
        ptx::tmem_st_32x32b_x16(tS + c * 16, pk);  // P (bf16 pairs) over the S columns
      }
      float ra, rb, rc, rd;
      f2unpack(rsv[0], ra, rb);
      f2unpack(rsv[1], rc, rd);
      const float rs = (ra + rb) + (rc + rd);
      l = l * f + rs;
      if (rescale && j > 0) {
#pragma unroll
        for (int c = 0; c < HD / 32; ++c) {
          uint32_t o[32];
          ptx::tmem_ld_32x32b_x32(tO + c * 32, o);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * f);
          ptx::tmem_st_32x32b_x32(tO + c * 32, o);
        }
      }
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      ptx::mbar_arrive(p_full(t));
    }
    const int qrow = row0 + qbt * BQ + r;
    if (p.kv_split > 1 && (t ? n[1] : n[0]) > 0) {
      // split-KV: this CTA's share, unnormalised (O relative to m_run, like l)
      float* op = p.opart + (static_cast<int64_t>(split) * p.T + qrow) * (p.heads * HD) + head * HD;
      float* ml = p.mlpart + ((static_cast<int64_t>(split) * p.T + qrow) * p.heads + head) * 2;
      if (nt > 0) {
        ptx::mbar_wait(o_done(t), 0);
        ptx::tc_fence_after();
      }
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {
        uint32_t u[32];
        if (nt > 0) {
          ptx::tmem_ld_32x32b_x32(tO + c * 32, u);
          ptx::tmem_wait_ld();
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) u[i] = 0u;
        }
#pragma unroll
        for (int v = 0; v < 8; ++v)
          reinterpret_cast<float4*>(op + c * 32)[v] = make_float4(__uint_as_float(u[4 * v]), __uint_as_float(u[4 * v + 1]),
                                                                 __uint_as_float(u[4 * v + 2]), __uint_as_float(u[4 * v + 3]));
      }
      ml[0] = nt > 0 ? m_run : -INFINITY;
      ml[1] = nt > 0 ? l : 0.f;
    } else if (nt > 0) {
      ptx::mbar_wait(o_done(t), 0);
      ptx::tc_fence_after();
      const float inv = 1.f / l;
      __nv_bfloat16* orow = p.ctx + static_cast<int64_t>(qrow) * p.ld_ctx + head * HD;
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {
        uint32_t u[32];
        ptx::tmem_ld_32x32b_x32(tO + c * 32, u);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(u[8 * v + 0]) * inv, __uint_as_float(u[8 * v + 1]) * inv);
          w.y = pack_bf16(__uint_as_float(u[8 * v + 2]) * inv, __uint_as_float(u[8 * v + 3]) * inv);
          w.z = pack_bf16(__uint_as_float(u[8 * v + 4]) * inv, __uint_as_float(u[8 * v + 5]) * inv);
          w.w = pack_bf16(__uint_as_float(u[8 * v + 6]) * inv, __uint_as_float(u[8 * v + 7]) * inv);
          *reinterpret_cast<uint4*>(orow + c * 32 + 8 * v) = w;
        }
      }
      p.lse[static_cast<int64_t>(head) * p.T + qrow] = (m_run + log2f(l)) * kLn2;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------- forward v3
// As v2 (two 128-row query tiles per CTA, P through TMEM, MMA ping-pong), but
// TWO softmax threads per query row: each tile has 8 softmax warps (warps
// 2-9: tile 0, 10-17: tile 1); warp w reads TMEM lane quadrant w % 4 and
// column half ((w - 2) % 8) / 4 of the score row.  The row max is combined
// through shared memory (one named barrier per tile and step, double-buffered
// by step parity); the row sums stay per half until the end.  Every SM
// sub-partition then runs two softmax warps per tile instead of one, so the
// exp / convert / TMEM-store chain of one warp hides behind the other's —
// v2's softmax ran at about half the MUFU rate with one warp per
// sub-partition.  The lazy-rescale decision is identical in both halves (same
// row maxima, same history).
constexpr int kFwd3Threads = 576;
constexpr int kFwd3Smem = 6 * kTile + 128 + 4096 + 1024;

__global__ void __launch_bounds__(kFwd3Threads, 1) attn_fwd3_kernel(const __grid_constant__ CUtensorMap tm_qkv, FwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  auto sQ = [&](int t) { return base + t * kTile; };
  auto sK = [&](int s) { return base + 2 * kTile + s * 2 * kTile; };
  auto sV = [&](int s) { return base + 3 * kTile + s * 2 * kTile; };
  const uint32_t bars = base + 6 * kTile;
  const uint32_t q_full = bars;
  auto kv_full = [&](int s) { return bars + 8 + 8 * s; };
  auto kv_empty = [&](int s) { return bars + 24 + 8 * s; };
  auto s_full = [&](int t) { return bars + 40 + 8 * t; };
  auto p_full = [&](int t) { return bars + 56 + 8 * t; };
  auto o_done = [&](int t) { return bars + 72 + 8 * t; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw + (bars + 88 - raw));
  // row-max exchange: [tile][parity][half][128 rows] fp32
  float* xbuf = reinterpret_cast<float*>(smem_raw + (bars + 128 - raw));

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nq = p.seq / BQ, nm = (nq + 1) / 2, nseq = p.T / p.seq;
  const int per = p.heads * nseq;
  int m, rest;
  cta_order(p.grouped, per, nm, m, rest);
  if (p.causal) m = nm - 1 - m;  // heaviest first
  const int head = rest % p.heads, sq = rest / p.heads;
  const int row0 = sq * p.seq;
  int qblk[2], n[2];
  for (int t = 0; t < 2; ++t) {
    qblk[t] = 2 * m + t;
    n[t] = qblk[t] < nq ? (p.causal ? qblk[t] + 1 : nq) : 0;
  }
  const int nkv = n[0] > n[1] ? n[0] : n[1];
  const int qcol = head * 3 * HD;

  if (threadIdx.x == 0) {
    ptx::mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(kv_full(s), 1);
      ptx::mbar_init(kv_empty(s), 1);
      ptx::mbar_init(s_full(s), 1);
      ptx::mbar_init(p_full(s), 256);
      ptx::mbar_init(o_done(s), 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc(ptx::smem_u32(tmem_slot), 512);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);

  if (warp == 0) {
    if (lane == 0) {
      ptx::prefetch_tmap(&tm_qkv);
      ptx::mbar_arrive_expect_tx(q_full, (n[1] > 0 ? 2 : 1) * kTile);
      for (int t = 0; t < 2; ++t) {
        if (n[t] == 0) continue;
        const int qr = row0 + qblk[t] * BQ;
        ptx::tma_load_2d(sQ(t), &tm_qkv, q_full, qcol, qr);
        ptx::tma_load_2d(sQ(t) + kHalf, &tm_qkv, q_full, qcol + 64, qr);
      }
      for (int j = 0; j < nkv; ++j) {
        const int s = j & 1;
        ptx::mbar_wait(kv_empty(s), ((j >> 1) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(kv_full(s), 2 * kTile);
        const int kr = row0 + j * BKV;
        ptx::tma_load_2d(sK(s), &tm_qkv, kv_full(s), qcol + HD, kr);
        ptx::tma_load_2d(sK(s) + kHalf, &tm_qkv, kv_full(s), qcol + HD + 64, kr);
        ptx::tma_load_2d(sV(s), &tm_qkv, kv_full(s), qcol + 2 * HD, kr);
        ptx::tma_load_2d(sV(s) + kHalf, &tm_qkv, kv_full(s), qcol + 2 * HD + 64, kr);
      }
    }
  } else if (warp == 1) {
    {  // identical to v2: the whole warp runs the issue loop, one elected lane issues
      constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(128, 128, 0, 0);
      constexpr uint32_t idesc_o = ptx::idesc_bf16_f32(128, 128, 0, 1);
      auto adv = [](uint64_t d, uint32_t bytes) { return d + (bytes >> 4); };
      const uint64_t q_kmaj[2] = {ptx::smem_desc_sw128(sQ(0), 16, 1024), ptx::smem_desc_sw128(sQ(1), 16, 1024)};
      const uint64_t k_kmaj[2] = {ptx::smem_desc_sw128(sK(0), 16, 1024), ptx::smem_desc_sw128(sK(1), 16, 1024)};
      const uint64_t v_mnmaj[2] = {ptx::smem_desc_sw128(sV(0), kHalf, 1024), ptx::smem_desc_sw128(sV(1), kHalf, 1024)};
      int kv_seen = -1;
      auto need_kv = [&](int j) {
        if (j > kv_seen) {
          ptx::mbar_wait(kv_full(j & 1), (j >> 1) & 1);
          ptx::tc_fence_after();
          kv_seen = j;
        }
      };
      auto issue_s = [&](int t, int j) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          ptx::mma_bf16_ss_w(tmem + 256 * t, adv(q_kmaj[t], (kk >> 2) * kHalf + (kk & 3) * 32),
                             adv(k_kmaj[j & 1], (kk >> 2) * kHalf + (kk & 3) * 32), idesc_s, kk > 0 ? 1u : 0u);
        ptx::mma_commit_w(s_full(t));
      };
      ptx::mbar_wait(q_full, 0);
      need_kv(0);
      for (int t = 0; t < 2; ++t)
        if (n[t] > 0) issue_s(t, 0);
      for (int j = 0; j < nkv; ++j) {
        for (int t = 0; t < 2; ++t) {
          if (j >= n[t]) continue;
          ptx::mbar_wait(p_full(t), j & 1);
          ptx::tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk)
            ptx::mma_bf16_ts_w(tmem + 256 * t + 128, tmem + 256 * t + kk * 8, adv(v_mnmaj[j & 1], kk * 2048), idesc_o,
                               (j | kk) != 0 ? 1u : 0u);
          if (j + 1 == n[t]) ptx::mma_commit_w(o_done(t));
          if (j + 1 < n[t]) {
            need_kv(j + 1);
            issue_s(t, j + 1);
          }
        }
        ptx::mma_commit_w(kv_empty(j & 1));
      }
    }
  } else {
    // ------------------------------------------------ softmax of tile t, row r, column half hf
    const int t = (warp - 2) / 8;
    const int hf = ((warp - 2) % 8) / 4;
    const int nt = t ? n[1] : n[0], qbt = t ? qblk[1] : qblk[0];
    const int q4 = warp % 4;  // TMEM lane quarter this warp may access
    const int r = q4 * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const uint32_t tS = tmem + lane_off + 256 * t, tO = tS + 128;
    constexpr int HC = BKV / 2;  // score columns per thread
    float m_run = -INFINITY, l = 0.f;
    for (int j = 0; j < nt; ++j) {
      ptx::mbar_wait(s_full(t), j & 1);
      ptx::tc_fence_after();
      uint32_t u[HC / 32][32];
#pragma unroll
      for (int c = 0; c < HC / 32; ++c) ptx::tmem_ld_32x32b_x32(tS + HC * hf + c * 32, u[c]);
      ptx::tmem_wait_ld();
      if (p.causal && j == qbt) {  // diagonal block: keys after the query row are masked
#pragma unroll
        for (int c = 0; c < HC; ++c)
          if (HC * hf + c > r) u[c / 32][c % 32] = __float_as_uint(-INFINITY);
      }
      float mx[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mx[i] = __uint_as_float(u[i / 32][i % 32]);
#pragma unroll
      for (int c = 8; c < HC; c += 2)
        mx[(c / 2) % 8] = fmax3(mx[(c / 2) % 8], __uint_as_float(u[c / 32][c % 32]), __uint_as_float(u[c / 32][c % 32 + 1]));
      float mb = fmaxf(fmax3(mx[0], mx[1], mx[2]), fmax3(fmax3(mx[3], mx[4], mx[5]), mx[6], mx[7]));
      // the other half's maximum (after this barrier every thread of the tile
      // has also finished reading S, so P may overwrite any S column)
      float* xb = xbuf + ((t * 2 + (j & 1)) * 2) * 128;
      xb[hf * 128 + r] = mb;
      ptx::named_bar_sync(1 + t, 256);
      mb = fmaxf(mb, xb[(hf ^ 1) * 128 + r]) * p.scale_log2;
      const bool rescale = __any_sync(0xffffffffu, mb > m_run + 8.f);
      float f = 1.f;
      if (rescale) {
        const float m_new = fmaxf(m_run, mb);
        f = ex2(m_run - m_new);
        m_run = m_new;
      }
      const uint64_t sc2 = f2pack(p.scale_log2, p.scale_log2), nm2 = f2pack(-m_run, -m_run);
      uint64_t rsv[2] = {f2pack(0.f, 0.f), f2pack(0.f, 0.f)};
#pragma unroll
      for (int c = 0; c < HC / 32; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float x0, x1;
          f2unpack(ffma2(f2pack(__uint_as_float(u[c][2 * i]), __uint_as_float(u[c][2 * i + 1])), sc2, nm2), x0, x1);
          const float e0 = ex2(x0), e1 = ex2(x1);
          rsv[i % 2] = fadd2(rsv[i % 2], f2pack(e0, e1));
          pk[i] = pack_bf16(e0, e1);
        }
        ptx::tmem_st_32x32b_x16(tS + HC / 2 * hf + c * 16, pk);  // P (bf16 pairs) of this half
      }
      float ra, rb, rc, rd;
      f2unpack(rsv[0], ra, rb);
      f2unpack(rsv[1], rc, rd);
      l = l * f + ((ra + rb) + (rc + rd));  // this half's partial row sum
      if (rescale && j > 0) {
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) {
          uint32_t o[32];
          ptx::tmem_ld_32x32b_x32(tO + (HD / 2) * hf + c * 32, o);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * f);
          ptx::tmem_st_32x32b_x32(tO + (HD / 2) * hf + c * 32, o);
        }
      }
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      ptx::mbar_arrive(p_full(t));
    }
    if (nt > 0) {
      // full row sum = both halves' partial sums (same rescale history)
      float* xb = xbuf + ((t * 2 + (nt & 1)) * 2) * 128;
      xb[hf * 128 + r] = l;
      ptx::named_bar_sync(1 + t, 256);
      l += xb[(hf ^ 1) * 128 + r];
      ptx::mbar_wait(o_done(t), 0);
      ptx::tc_fence_after();
      const float inv = 1.f / l;
      const int qrow = row0 + qbt * BQ + r;
      __nv_bfloat16* orow = p.ctx + static_cast<int64_t>(qrow) * p.ld_ctx + head * HD + (HD / 2) * hf;
#pragma unroll
      for (int c = 0; c < HD / 64; ++c) {
        uint32_t u[32];
        ptx::tmem_ld_32x32b_x32(tO + (HD / 2) * hf + c * 32, u);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(u[8 * v + 0]) * inv, __uint_as_float(u[8 * v + 1]) * inv);
          w.y = pack_bf16(__uint_as_float(u[8 * v + 2]) * inv, __uint_as_float(u[8 * v + 3]) * inv);
          w.z = pack_bf16(__uint_as_float(u[8 * v + 4]) * inv, __uint_as_float(u[8 * v + 5]) * inv);
          w.w = pack_bf16(__uint_as_float(u[8 * v + 6]) * inv, __uint_as_float(u[8 * v + 7]) * inv);
          *reinterpret_cast<uint4*>(orow + c * 32 + 8 * v) = w;
        }
      }
      if (hf == 0) p.lse[static_cast<int64_t>(head) * p.T + qrow] = (m_run + log2f(l)) * kLn2;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------- forward v4
// v2 made persistent with Blackwell cluster launch control (CLC): the grid
// is still one CTA per query-tile pair (heaviest first), but a running CTA
// takes over not-yet-launched CTAs (`clusterlaunchcontrol.try_cancel`)
// instead of exiting, so barrier init, TMEM allocation and the tensor-map
// prefetch happen once per SM, the next item's Q / first K,V tiles load while
// the current item's last steps run, and its first S MMA overlaps the O
// drain.  The producer requests the successor with each item's last K/V
// load (late enough that the CTAs finishing first take the next items, as
// the hardware scheduler would); every role reads the 16-byte response from a two-slot ring
// (clc_full / clc_empty).  Barrier phases run across items (per-tile step,
// Q and O counters; one K/V ring counter).  kv_split == 1 only.
struct FwdItem {
  int qblk[2], nl[2], nkv, head, row0;
};

__device__ __forceinline__ FwdItem fwd_item(const FwdParams& p, int b) {
  FwdItem I;
  const int nq = p.seq / BQ, nm = (nq + 1) / 2, nseq = p.T / p.seq;
  int m, rest;
  cta_order(p.grouped, p.heads * nseq, nm, m, rest, b);
  if (p.causal) m = nm - 1 - m;
  I.head = rest % p.heads;
  I.row0 = (rest / p.heads) * p.seq;
  for (int t = 0; t < 2; ++t) {
    I.qblk[t] = 2 * m + t;
    I.nl[t] = I.qblk[t] < nq ? (p.causal ? I.qblk[t] + 1 : nq) : 0;
  }
  I.nkv = I.nl[0] > I.nl[1] ? I.nl[0] : I.nl[1];
  return I;
}

__device__ __forceinline__ void clc_try_cancel(uint32_t resp, uint32_t bar) {
  asm volatile("clusterlaunchcontrol.try_cancel.async.shared::cta.mbarrier::complete_tx::bytes.b128 [%0], [%1];" ::"r"(
                   resp),
               "r"(bar)
               : "memory");
}
// The stolen CTA's blockIdx.x, or -1 when no CTA was left to take.
__device__ __forceinline__ int clc_next(uint32_t resp) {
  uint32_t ok, x;
  asm volatile(
      "{\n\t.reg .b128 r;\n\t.reg .pred p;\n\t"
      "ld.shared.b128 r, [%2];\n\t"
      "clusterlaunchcontrol.query_cancel.is_canceled.pred.b128 p, r;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t"
      "@p clusterlaunchcontrol.query_cancel.get_first_ctaid::x.b32.b128 %1, r;\n\t}"
      : "=r"(ok), "=r"(x)
      : "r"(resp)
      : "memory");
  return ok ? static_cast<int>(x) : -1;
}

constexpr int kFwd4Smem = 6 * kTile + 256 + 1024;

__global__ void __launch_bounds__(320, 1) attn_fwd4_kernel(const __grid_constant__ CUtensorMap tm_qkv, FwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  auto sQ = [&](int t) { return base + t * kTile; };
  auto sK = [&](int s) { return base + 2 * kTile + s * 2 * kTile; };
  auto sV = [&](int s) { return base + 3 * kTile + s * 2 * kTile; };
  const uint32_t bars = base + 6 * kTile;
  auto kv_full = [&](int s) { return bars + 8 * s; };
  auto kv_empty = [&](int s) { return bars + 16 + 8 * s; };
  auto s_full = [&](int t) { return bars + 32 + 8 * t; };
  auto p_full = [&](int t) { return bars + 48 + 8 * t; };
  auto o_done = [&](int t) { return bars + 64 + 8 * t; };
  auto q_full = [&](int t) { return bars + 80 + 8 * t; };
  auto q_empty = [&](int t) { return bars + 96 + 8 * t; };
  auto clc_full = [&](int s) { return bars + 112 + 8 * s; };
  auto clc_empty = [&](int s) { return bars + 128 + 8 * s; };
  auto clc_resp = [&](int s) { return bars + 160 + 16 * s; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw + (bars + 144 - raw));

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(kv_full(s), 1);
      ptx::mbar_init(kv_empty(s), 1);
      ptx::mbar_init(s_full(s), 1);
      ptx::mbar_init(p_full(s), 128);
      ptx::mbar_init(o_done(s), 1);
      ptx::mbar_init(q_full(s), 1);
      ptx::mbar_init(q_empty(s), 1);
      ptx::mbar_init(clc_full(s), 1);
      ptx::mbar_init(clc_empty(s), 9);  // the MMA warp + 8 softmax warps
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc(ptx::smem_u32(tmem_slot), 512);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);

  if (warp == 0) {
    if (lane == 0) {
      ptx::prefetch_tmap(&tm_qkv);
      int qc[2] = {0, 0}, g = 0;
      for (int b = static_cast<int>(blockIdx.x), it = 0; b >= 0; ++it) {
        const FwdItem I = fwd_item(p, b);
        const int qcol = I.head * 3 * HD;
        for (int t = 0; t < 2; ++t) {
          if (I.nl[t] == 0) continue;
          ptx::mbar_wait(q_empty(t), (qc[t] & 1) ^ 1);
          ++qc[t];
          ptx::mbar_arrive_expect_tx(q_full(t), kTile);
          const int qr = I.row0 + I.qblk[t] * BQ;
          ptx::tma_load_2d(sQ(t), &tm_qkv, q_full(t), qcol, qr);
          ptx::tma_load_2d(sQ(t) + kHalf, &tm_qkv, q_full(t), qcol + 64, qr);
        }
        for (int j = 0; j < I.nkv; ++j, ++g) {
          const int s = g & 1;
          ptx::mbar_wait(kv_empty(s), ((g >> 1) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(kv_full(s), 2 * kTile);
          const int kr = I.row0 + j * BKV;
          ptx::tma_load_2d(sK(s), &tm_qkv, kv_full(s), qcol + HD, kr);
          ptx::tma_load_2d(sK(s) + kHalf, &tm_qkv, kv_full(s), qcol + HD + 64, kr);
          ptx::tma_load_2d(sV(s), &tm_qkv, kv_full(s), qcol + 2 * HD, kr);
          ptx::tma_load_2d(sV(s) + kHalf, &tm_qkv, kv_full(s), qcol + 2 * HD + 64, kr);
          if (j + 1 == I.nkv) {
            // ask for the successor item with the last K/V load (the MMA is ~2 steps
            // behind): claiming earlier would bind work to a CTA before it is known to
            // finish early (at s = 8192 a claim at the first load made the heaviest
            // items' CTAs take a second item: 0.12 -> 0.17 ms).  The slot's readers
            // are done with item it - 2.
            const int cs = it & 1;
            ptx::mbar_wait(clc_empty(cs), ((it >> 1) & 1) ^ 1);
            ptx::fence_proxy_async();
            ptx::mbar_arrive_expect_tx(clc_full(cs), 16);
            clc_try_cancel(clc_resp(cs), clc_full(cs));
          }
        }
        ptx::mbar_wait(clc_full(it & 1), (it >> 1) & 1);
        b = clc_next(clc_resp(it & 1));
      }
    }
  } else if (warp == 1) {
    // the whole warp runs the issue loop; each tcgen05 op is issued by one elected lane
    constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(128, 128, 0, 0);
    constexpr uint32_t idesc_o = ptx::idesc_bf16_f32(128, 128, 0, 1);
    auto adv = [](uint64_t d, uint32_t bytes) { return d + (bytes >> 4); };
    const uint64_t q_kmaj[2] = {ptx::smem_desc_sw128(sQ(0), 16, 1024), ptx::smem_desc_sw128(sQ(1), 16, 1024)};
    const uint64_t k_kmaj[2] = {ptx::smem_desc_sw128(sK(0), 16, 1024), ptx::smem_desc_sw128(sK(1), 16, 1024)};
    const uint64_t v_mnmaj[2] = {ptx::smem_desc_sw128(sV(0), kHalf, 1024), ptx::smem_desc_sw128(sV(1), kHalf, 1024)};
    int qc[2] = {0, 0}, sc[2] = {0, 0}, g0 = 0, kv_seen = -1;
    auto need_kv = [&](int gj) {  // global K/V block counter
      if (gj > kv_seen) {
        ptx::mbar_wait(kv_full(gj & 1), (gj >> 1) & 1);
        ptx::tc_fence_after();
        kv_seen = gj;
      }
    };
    auto issue_s = [&](int t, int gj) {
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk)
        ptx::mma_bf16_ss_w(tmem + 256 * t, adv(q_kmaj[t], (kk >> 2) * kHalf + (kk & 3) * 32),
                           adv(k_kmaj[gj & 1], (kk >> 2) * kHalf + (kk & 3) * 32), idesc_s, kk > 0 ? 1u : 0u);
      ptx::mma_commit_w(s_full(t));
    };
    for (int b = static_cast<int>(blockIdx.x), it = 0; b >= 0; ++it) {
      const FwdItem I = fwd_item(p, b);
      need_kv(g0);
      for (int t = 0; t < 2; ++t) {
        if (I.nl[t] == 0) continue;
        ptx::mbar_wait(q_full(t), qc[t] & 1);
        ++qc[t];
        ptx::tc_fence_after();
        issue_s(t, g0);
        if (I.nl[t] == 1) ptx::mma_commit_w(q_empty(t));
      }
      for (int j = 0; j < I.nkv; ++j) {  // tile t is active for j < nl[t]
        for (int t = 0; t < 2; ++t) {
          if (j >= I.nl[t]) continue;
          ptx::mbar_wait(p_full(t), sc[t] & 1);
          ++sc[t];
          ptx::tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk)
            ptx::mma_bf16_ts_w(tmem + 256 * t + 128, tmem + 256 * t + kk * 8, adv(v_mnmaj[(g0 + j) & 1], kk * 2048),
                               idesc_o, (j | kk) != 0 ? 1u : 0u);
          if (j + 1 == I.nl[t]) ptx::mma_commit_w(o_done(t));
          if (j + 1 < I.nl[t]) {
            need_kv(g0 + j + 1);
            issue_s(t, g0 + j + 1);
            if (j + 2 == I.nl[t]) ptx::mma_commit_w(q_empty(t));  // last S of this tile: Q may be replaced
          }
        }
        ptx::mma_commit_w(kv_empty((g0 + j) & 1));
      }
      g0 += I.nkv;
      ptx::mbar_wait(clc_full(it & 1), (it >> 1) & 1);
      b = clc_next(clc_resp(it & 1));
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(clc_empty(it & 1));
    }
  } else {
    // ------------------------------------------------ softmax of tile t, row r (as v2)
    const int t = (warp - 2) / 4;
    const int q4 = warp % 4;  // TMEM lane quarter this warp may access
    const int r = q4 * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const uint32_t tS = tmem + lane_off + 256 * t, tO = tS + 128;
    int sc = 0, oc = 0;
    for (int b = static_cast<int>(blockIdx.x), it = 0; b >= 0; ++it) {
      const FwdItem I = fwd_item(p, b);
      const int nt = I.nl[t], qbt = I.qblk[t];
      float m_run = -INFINITY, l = 0.f;
      for (int j = 0; j < nt; ++j, ++sc) {
        ptx::mbar_wait(s_full(t), sc & 1);
        ptx::tc_fence_after();
        uint32_t u[BKV / 32][32];
#pragma unroll
        for (int c = 0; c < BKV / 32; ++c) ptx::tmem_ld_32x32b_x32(tS + c * 32, u[c]);
        ptx::tmem_wait_ld();
        if (p.causal && j == qbt) {
#pragma unroll
          for (int c = 0; c < BKV; ++c)
            if (c > r) u[c / 32][c % 32] = __float_as_uint(-INFINITY);
        }
        float mx[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) mx[i] = __uint_as_float(u[i / 32][i % 32]);
#pragma unroll
        for (int c = 8; c < BKV; c += 2)
          mx[(c / 2) % 8] = fmax3(mx[(c / 2) % 8], __uint_as_float(u[c / 32][c % 32]), __uint_as_float(u[c / 32][c % 32 + 1]));
        float mb = fmaxf(fmax3(mx[0], mx[1], mx[2]), fmax3(fmax3(mx[3], mx[4], mx[5]), mx[6], mx[7]));
        mb *= p.scale_log2;
        const bool rescale = __any_sync(0xffffffffu, mb > m_run + 8.f);
        float f = 1.f;
        if (rescale) {
          const float m_new = fmaxf(m_run, mb);
          f = ex2(m_run - m_new);
          m_run = m_new;
        }
        const uint64_t sc2 = f2pack(p.scale_log2, p.scale_log2), nm2 = f2pack(-m_run, -m_run);
        uint64_t rsv[2] = {f2pack(0.f, 0.f), f2pack(0.f, 0.f)};
#pragma unroll
        for (int c = 0; c < BKV / 32; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float x0, x1;
            f2unpack(ffma2(f2pack(__uint_as_float(u[c][2 * i]), __uint_as_float(u[c][2 * i + 1])), sc2, nm2), x0, x1);
            const float e0 = ex2(x0), e1 = ex2(x1);
            rsv[i % 2] = fadd2(rsv[i % 2], f2pack(e0, e1));
            pk[i] = pack_bf16(e0, e1);
          }
          ptx::tmem_st_32x32b_x16(tS + c * 16, pk);
        }
        float ra, rb, rc, rd;
        f2unpack(rsv[0], ra, rb);
        f2unpack(rsv[1], rc, rd);
        l = l * f + ((ra + rb) + (rc + rd));
        if (rescale && j > 0) {
#pragma unroll
          for (int c = 0; c < HD / 32; ++c) {
            uint32_t o[32];
            ptx::tmem_ld_32x32b_x32(tO + c * 32, o);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * f);
            ptx::tmem_st_32x32b_x32(tO + c * 32, o);
          }
        }
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        ptx::mbar_arrive(p_full(t));
      }
      if (nt > 0) {
        ptx::mbar_wait(o_done(t), oc & 1);
        ++oc;
        ptx::tc_fence_after();
        const int qrow = I.row0 + qbt * BQ + r;
        const float inv = 1.f / l;
        __nv_bfloat16* orow = p.ctx + static_cast<int64_t>(qrow) * p.ld_ctx + I.head * HD;
#pragma unroll
        for (int c = 0; c < HD / 32; ++c) {
          uint32_t u[32];
          ptx::tmem_ld_32x32b_x32(tO + c * 32, u);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            uint4 w;
            w.x = pack_bf16(__uint_as_float(u[8 * v + 0]) * inv, __uint_as_float(u[8 * v + 1]) * inv);
            w.y = pack_bf16(__uint_as_float(u[8 * v + 2]) * inv, __uint_as_float(u[8 * v + 3]) * inv);
            w.z = pack_bf16(__uint_as_float(u[8 * v + 4]) * inv, __uint_as_float(u[8 * v + 5]) * inv);
            w.w = pack_bf16(__uint_as_float(u[8 * v + 6]) * inv, __uint_as_float(u[8 * v + 7]) * inv);
            *reinterpret_cast<uint4*>(orow + c * 32 + 8 * v) = w;
          }
        }
        p.lse[static_cast<int64_t>(I.head) * p.T + qrow] = (m_run + log2f(l)) * kLn2;
        ptx::tc_fence_before();  // the O reads complete before the next item's PV (ordered by p_full)
      }
      ptx::mbar_wait(clc_full(it & 1), (it >> 1) & 1);
      b = clc_next(clc_resp(it & 1));
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(clc_empty(it & 1));
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// ================================================================ backward
// dV = P^T dO, dP = dO V^T, dS = P * (dP - D) with D = rowsum(dO * O),
// dQ = dS K / sqrt(d), dK = dS^T Q / sqrt(d)   (FlashAttention-2 order).
// One CTA per (128-key block, head, sequence) loops over the query blocks that
// see it; TMEM: S (reused for the dQ tile) [0,128), dP [128,256), dV
// [256,384), dK [384,512).  P and dS (bf16) are written once to shared memory
// in the SW128 layout [query rows][key cols]: the same bytes are the K-major A
// operand of dQ = dS K and the MN-major A operand of dV = P^T dO / dK = dS^T Q.
// dQ tiles are added to an fp32 accumulator with vector atomics; a finalize
// kernel scales and converts them.
struct BwdParams {
  int T, seq, heads, causal;
  int grouped;  // as FwdParams::grouped
  float scale_log2;  // log2(e) / sqrt(d)
  float scale;       // 1 / sqrt(d)
  const float* lse;  // [heads][T] natural log (forward output)
  const float* D;    // [heads][T] rowsum(dO * O)
  float* dq_acc;     // [T][heads*128] fp32
  __nv_bfloat16* dqkv;
  int64_t ld_dqkv;
};

__global__ void __launch_bounds__(320, 1) attn_bwd_kernel(const __grid_constant__ CUtensorMap tm_qkv,
                                                          const __grid_constant__ CUtensorMap tm_do,
                                                          const __grid_constant__ CUtensorMap tm_dq, BwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t sK = base, sV = base + kTile, sQ = base + 2 * kTile, sdO = base + 3 * kTile;
  const uint32_t sP = base + 4 * kTile, sdS = base + 5 * kTile;
  const uint32_t bars = base + 6 * kTile;
  const uint32_t kv_full = bars, qdo_full = bars + 8, qdo_empty = bars + 16, s_full = bars + 24;
  const uint32_t ds_full = bars + 32, dq_full = bars + 40, s_free = bars + 48, done = bars + 56;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw + (bars + 64 - raw));

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nkb = p.seq / BKV, nseq = p.T / p.seq, per = p.heads * nseq;
  const int jb = static_cast<int>(blockIdx.x) / per;  // causal: key block 0 sees the most query blocks
  const int rest = static_cast<int>(blockIdx.x) % per;
  const int head = rest % p.heads, sq = rest / p.heads;
  const int row0 = sq * p.seq, kvrow = row0 + jb * BKV;
  const int i0 = p.causal ? jb : 0, n = nkb - i0;
  const int qcol = head * 3 * HD;

  if (threadIdx.x == 0) {
    ptx::mbar_init(kv_full, 1);
    ptx::mbar_init(qdo_full, 1);
    ptx::mbar_init(qdo_empty, 1);
    ptx::mbar_init(s_full, 1);
    ptx::mbar_init(ds_full, 256);
    ptx::mbar_init(dq_full, 1);
    ptx::mbar_init(s_free, 256);
    ptx::mbar_init(done, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc(ptx::smem_u32(tmem_slot), 512);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);

  if (warp == 0) {
    if (lane == 0) {
      ptx::prefetch_tmap(&tm_qkv);
      ptx::prefetch_tmap(&tm_do);
      ptx::mbar_arrive_expect_tx(kv_full, 2 * kTile);
      ptx::tma_load_2d(sK, &tm_qkv, kv_full, qcol + HD, kvrow);
      ptx::tma_load_2d(sK + kHalf, &tm_qkv, kv_full, qcol + HD + 64, kvrow);
      ptx::tma_load_2d(sV, &tm_qkv, kv_full, qcol + 2 * HD, kvrow);
      ptx::tma_load_2d(sV + kHalf, &tm_qkv, kv_full, qcol + 2 * HD + 64, kvrow);
      for (int t = 0; t < n; ++t) {
        const int qr = row0 + (i0 + t) * BQ;
        ptx::mbar_wait(qdo_empty, (t & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(qdo_full, 2 * kTile);
        ptx::tma_load_2d(sQ, &tm_qkv, qdo_full, qcol, qr);
        ptx::tma_load_2d(sQ + kHalf, &tm_qkv, qdo_full, qcol + 64, qr);
        ptx::tma_load_2d(sdO, &tm_do, qdo_full, head * HD, qr);
        ptx::tma_load_2d(sdO + kHalf, &tm_do, qdo_full, head * HD + 64, qr);
      }
      ptx::mbar_wait(qdo_empty, (n & 1) ^ 1);  // tail: the last Q/dO tile released
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_kk = ptx::idesc_bf16_f32(128, 128, 0, 0);  // both K-major
      constexpr uint32_t id_mm = ptx::idesc_bf16_f32(128, 128, 1, 1);  // both MN-major
      constexpr uint32_t id_km = ptx::idesc_bf16_f32(128, 128, 0, 1);  // A K-major, B MN-major
      ptx::mbar_wait(kv_full, 0);
      for (int t = 0; t < n; ++t) {
        ptx::mbar_wait(qdo_full, t & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)  // S = Q K^T
          ptx::mma_bf16_ss(tmem, desc_kmajor(sQ, kk), desc_kmajor(sK, kk), id_kk, kk > 0 ? 1u : 0u);
        if (t > 0) {
          ptx::mbar_wait(s_free, (t - 1) & 1);  // dQ tile of t-1 read out of the dP columns
          ptx::tc_fence_after();
        }
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)  // dP = dO V^T
          ptx::mma_bf16_ss(tmem + 128, desc_kmajor(sdO, kk), desc_kmajor(sV, kk), id_kk, kk > 0 ? 1u : 0u);
        ptx::mma_commit(s_full);
        ptx::mbar_wait(ds_full, t & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < BQ / 16; ++kk)  // dV += P^T dO
          ptx::mma_bf16_ss(tmem + 256, desc_mnmajor(sP, kk), desc_mnmajor(sdO, kk), id_mm, (t | kk) != 0 ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < BQ / 16; ++kk)  // dK += dS^T Q
          ptx::mma_bf16_ss(tmem + 384, desc_mnmajor(sdS, kk), desc_mnmajor(sQ, kk), id_mm, (t | kk) != 0 ? 1u : 0u);
        ptx::mma_commit(qdo_empty);  // Q and dO of t are no longer read: the next load can start
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk)  // dQ tile = dS K (into the dP columns)
          ptx::mma_bf16_ss(tmem + 128, desc_kmajor(sdS, kk), desc_mnmajor(sK, kk), id_km, kk > 0 ? 1u : 0u);
        ptx::mma_commit(dq_full);
      }
      ptx::mma_commit(done);
      if (n > 0) ptx::mbar_wait(s_free, (n - 1) & 1);  // tail: the last dQ tile read out
    }
  } else {
    // ---- warps 2-9: two threads per query row, columns [64*half, 64*half + 64)
    const int half = (warp - 2) / 4, q4 = warp % 4;
    const int r = q4 * 32 + lane, c0 = 64 * half;
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const int ldq = p.heads * HD;
    for (int t = 0; t < n; ++t) {
      const int i = i0 + t;
      const int qrow = row0 + i * BQ + r;
      const float lse2 = p.lse[static_cast<int64_t>(head) * p.T + qrow] * 1.4426950408889634f;
      const float Dr = p.D[static_cast<int64_t>(head) * p.T + qrow];
      ptx::mbar_wait(s_full, t & 1);
      ptx::tc_fence_after();
      uint32_t su[2][32], du[2][32];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        ptx::tmem_ld_32x32b_x32(tmem + lane_off + c0 + 32 * c, su[c]);
        ptx::tmem_ld_32x32b_x32(tmem + lane_off + 128 + c0 + 32 * c, du[c]);
      }
      ptx::tmem_wait_ld();
      const bool diag = p.causal && i == jb;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        float pv[32], ds[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const float e = ex2(fmaf(__uint_as_float(su[c][k]), p.scale_log2, -lse2));
          pv[k] = (diag && c0 + 32 * c + k > r) ? 0.f : e;
          ds[k] = pv[k] * (__uint_as_float(du[c][k]) - Dr);
        }
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int c16 = (c0 + 32 * c) / 8 + v;
          st_shared_v4(sP + sw128_off(r, c16), pack_bf16(pv[8 * v], pv[8 * v + 1]), pack_bf16(pv[8 * v + 2], pv[8 * v + 3]),
                       pack_bf16(pv[8 * v + 4], pv[8 * v + 5]), pack_bf16(pv[8 * v + 6], pv[8 * v + 7]));
          st_shared_v4(sdS + sw128_off(r, c16), pack_bf16(ds[8 * v], ds[8 * v + 1]), pack_bf16(ds[8 * v + 2], ds[8 * v + 3]),
                       pack_bf16(ds[8 * v + 4], ds[8 * v + 5]), pack_bf16(ds[8 * v + 6], ds[8 * v + 7]));
        }
      }
      ptx::fence_proxy_async();
      ptx::tc_fence_before();
      ptx::mbar_arrive(ds_full);
      // dQ tile (unscaled) -> fp32 accumulator with one TMA bulk reduce-add per
      // 32-column box: the tile is staged (SW128, conflict-free) in the P/dS
      // region, free once the dQ MMA that read it has completed.
      ptx::mbar_wait(dq_full, t & 1);
      ptx::tc_fence_after();
      uint32_t qu[2][32];
#pragma unroll
      for (int c = 0; c < 2; ++c) ptx::tmem_ld_32x32b_x32(tmem + lane_off + 128 + c0 + 32 * c, qu[c]);
      ptx::tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const uint32_t box = sP + static_cast<uint32_t>((c0 + 32 * c) / 32) * kHalf;  // [128 rows][32 fp32]
#pragma unroll
        for (int v = 0; v < 8; ++v)
          st_shared_v4(box + r * 128 + ((v ^ (r & 7)) << 4), qu[c][4 * v], qu[c][4 * v + 1], qu[c][4 * v + 2],
                       qu[c][4 * v + 3]);
      }
      ptx::fence_proxy_async();
      ptx::named_bar_sync(1, 256);
      if (warp == 2 && lane == 0) {
#pragma unroll
        for (int b = 0; b < 4; ++b) ptx::tma_reduce_add_2d(&tm_dq, sP + b * kHalf, head * HD + 32 * b, row0 + i * BQ);
        ptx::bulk_commit();
        ptx::bulk_wait_read0();  // staging may be overwritten (next P/dS) only after the reads
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(s_free);
    }
    if (warp == 2 && lane == 0) ptx::bulk_wait0();  // reductions complete before the dQ finalize kernel
    // ---- dK (scaled), dV -> dqkv rows of this key block (TMEM lane = key row)
    ptx::mbar_wait(done, 0);
    ptx::tc_fence_after();
    __nv_bfloat16* drow = p.dqkv + static_cast<int64_t>(kvrow + r) * p.ld_dqkv + qcol;
#pragma unroll
    for (int which = 0; which < 2; ++which) {  // 0: dK, 1: dV
      const float f = which == 0 ? p.scale : 1.f;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t u[32];
        ptx::tmem_ld_32x32b_x32(tmem + lane_off + (which == 0 ? 384 : 256) + c0 + 32 * c, u);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(u[8 * v + 0]) * f, __uint_as_float(u[8 * v + 1]) * f);
          w.y = pack_bf16(__uint_as_float(u[8 * v + 2]) * f, __uint_as_float(u[8 * v + 3]) * f);
          w.z = pack_bf16(__uint_as_float(u[8 * v + 4]) * f, __uint_as_float(u[8 * v + 5]) * f);
          w.w = pack_bf16(__uint_as_float(u[8 * v + 6]) * f, __uint_as_float(u[8 * v + 7]) * f);
          *reinterpret_cast<uint4*>(drow + (which == 0 ? HD : 2 * HD) + c0 + 32 * c + 8 * v) = w;
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------- backward v2
// Transposed formulation, 64-query blocks, tensor core and softmax overlapped
// (default; ATP_ATTN_BWD=1 selects v1 above).  One CTA per (128-key block j,
// head, sequence) loops over the 64-row query blocks i that see it.  Keys are
// the TMEM lanes of every product:
//   S^T  = K Q_i^T        [128 keys][64 q]   (A = K K-major,  B = Q_i K-major)
//   dP^T = V dO_i^T       [128 keys][64 q]   (A = V K-major,  B = dO_i K-major)
//   P^T  = exp2(S^T c - lse_q),  dS^T = P^T * (dP^T - D_q)   (softmax warps, lane = key)
//   dV  += P^T dO_i       [128 keys][128 d]  (A = P^T from TMEM, B = dO_i MN-major)
//   dK  += dS^T Q_i       [128 keys][128 d]  (A = dS^T from TMEM, B = Q_i MN-major)
//   dQ_i^T = K^T dS^T     [128 d][64 q]      (A = K MN-major, B = dS^T MN-major) -> fp32
//            accumulator with a TMA bulk reduce-add by four dQ warps.
// TMEM: S^T and dP^T double-buffered (2 x 64 + 2 x 64 columns), dV and dK 2 x
// 128.  The softmax writes P^T and dS^T (bf16 pairs) over the S^T / dP^T
// columns it read (dS^T also to shared memory, the B operand of dQ^T), and
// dQ_i^T goes into the dP^T buffer of its block, issued after dK read it.
// The MMA warp issues S^T / dP^T of block i+1 before waiting for the softmax of
// block i, so the tensor core works on the next block while the softmax warps
// run; dQ readout has its own warps.  Q_i, dO_i (+ lse, D) sit in a 3-deep TMA
// ring (the load of block i+3 starts when dK of block i is done: one block of
// slack for the load latency), dS^T is double-buffered: 226 KB of shared memory.
// Warps: 0 TMA, 1 MMA, 2-9 softmax (lane quadrant w%4, 32 query columns each),
// 10-13 dQ readout (d quadrant w%4); the 8 softmax warps then drain dK / dV.
// Measured (b4 s2048 32 heads causal): 0.63 ms vs 0.71 ms for v1; shared-memory
// traffic (~300 KB per 64-query block) is what bounds it now.
constexpr int BQ2 = 64;
constexpr uint32_t kQ2 = BQ2 * 128 * 2;     // [64 rows][128 cols] bf16 = 16 KB (two 8 KB SW128 boxes)
constexpr uint32_t kBox64 = BQ2 * 128;      // one [64 rows][64 cols] bf16 SW128 box = 8 KB
constexpr uint32_t kPS = 128 * BQ2 * 2;     // [128 keys][64 q] bf16 = 16 KB (one SW128 box)
constexpr uint32_t kDqBox = BQ2 * 32 * 4;   // [64 q][32 d] fp32 = 8 KB (SW128)
constexpr int kQSlots = 3;  // Q_i / dO_i (+ lse, D) ring depth: covers the TMA latency of block i+3
struct Bwd2Smem {
  static constexpr uint32_t K = 0, V = kTile, Q = 2 * kTile;  // Q[3], then dO[3]
  static constexpr uint32_t dO = Q + kQSlots * kQ2;
  static constexpr uint32_t dS = dO + kQSlots * kQ2;  // dS^T[2]
  static constexpr uint32_t dQ = dS + 2 * kPS;        // 4 boxes [64 q][32 d] fp32
  static constexpr uint32_t LD = dQ + 4 * kDqBox;     // lse[3][64], D[3][64] fp32
  static constexpr uint32_t Bars = LD + 2 * kQSlots * BQ2 * 4;
  static constexpr uint32_t Bytes = Bars + 256 + 1024;
};
static_assert(Bwd2Smem::Bytes <= 232448, "attention backward v2: shared memory");

__device__ __forceinline__ uint64_t desc_k64(uint32_t tile, int kk) {  // [64 rows][128 K] K-major, 2 boxes
  return ptx::smem_desc_sw128(tile + (kk >> 2) * kBox64 + (kk & 3) * 32, 16, 1024);
}
__device__ __forceinline__ uint64_t desc_mn64(uint32_t tile, int kk) {  // [64 K rows][128 MN] MN-major, 2 boxes
  return ptx::smem_desc_sw128(tile + kk * 2048, kBox64, 1024);
}
__device__ __forceinline__ uint64_t desc_k_ps(uint32_t tile, int kk) {  // [128 rows][64 K] K-major, 1 box
  return ptx::smem_desc_sw128(tile + kk * 32, 16, 1024);
}
__device__ __forceinline__ uint64_t desc_mn_ps(uint32_t tile, int kk) {  // [128 K rows][64 MN] MN-major, 1 box
  return ptx::smem_desc_sw128(tile + kk * 2048, kPS, 1024);
}

__global__ void __launch_bounds__(448, 1) attn_bwd2_kernel(const __grid_constant__ CUtensorMap tm_kv,
                                                           const __grid_constant__ CUtensorMap tm_q,
                                                           const __grid_constant__ CUtensorMap tm_do,
                                                           const __grid_constant__ CUtensorMap tm_dq, BwdParams p) {
  using L = Bwd2Smem;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const float* lds = reinterpret_cast<const float*>(smem_raw + (base - raw) + L::LD);  // lse[3][64], D[3][64]
  const uint32_t bars = base + L::Bars;
  const uint32_t kv_full = bars;
  auto q_full = [&](int q) { return bars + 8 + 8 * q; };    // [3]
  auto q_empty = [&](int q) { return bars + 32 + 8 * q; };  // [3]
  auto s_full = [&](int s) { return bars + 56 + 8 * s; };
  auto ds_full = [&](int s) { return bars + 72 + 8 * s; };
  auto p_free = [&](int s) { return bars + 88 + 8 * s; };
  auto dq_full = [&](int s) { return bars + 104 + 8 * s; };
  auto s_free = [&](int s) { return bars + 120 + 8 * s; };
  const uint32_t done = bars + 136;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw + (bars + 144 - raw));

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nseq = p.T / p.seq, per = p.heads * nseq, nkb = p.seq / BKV;
  int jb, rest;  // causal: key block 0 sees the most query blocks
  cta_order(p.grouped, per, nkb, jb, rest);
  const int head = rest % p.heads, sq = rest / p.heads;
  const int row0 = sq * p.seq, kvrow = row0 + jb * BKV;
  const int nqb = p.seq / BQ2;
  const int i0 = p.causal ? 2 * jb : 0, n = nqb - i0;
  const int qcol = head * 3 * HD;

  if (threadIdx.x == 0) {
    ptx::mbar_init(kv_full, 1);
    for (int q = 0; q < kQSlots; ++q) {
      ptx::mbar_init(q_full(q), 1);
      ptx::mbar_init(q_empty(q), 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(s_full(s), 1);
      ptx::mbar_init(ds_full(s), 256);
      ptx::mbar_init(p_free(s), 1);
      ptx::mbar_init(dq_full(s), 1);
      ptx::mbar_init(s_free(s), 128);
    }
    ptx::mbar_init(done, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc(ptx::smem_u32(tmem_slot), 512);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);
  // TMEM columns: S^T[s] (then P^T bf16 pairs in its columns [0,16) and [32,48)),
  // dP^T[s] (then dQ^T of the same block), dV, dK.
  auto tS = [&](int s) { return tmem + 64u * s; };
  auto tdP = [&](int s) { return tmem + 128u + 64u * s; };
  const uint32_t tdV = tmem + 256, tdK = tmem + 384;

  if (warp == 0) {
    if (lane == 0) {
      ptx::prefetch_tmap(&tm_kv);
      ptx::prefetch_tmap(&tm_q);
      ptx::prefetch_tmap(&tm_do);
      ptx::mbar_arrive_expect_tx(kv_full, 2 * kTile);
      ptx::tma_load_2d(base + L::K, &tm_kv, kv_full, qcol + HD, kvrow);
      ptx::tma_load_2d(base + L::K + kHalf, &tm_kv, kv_full, qcol + HD + 64, kvrow);
      ptx::tma_load_2d(base + L::V, &tm_kv, kv_full, qcol + 2 * HD, kvrow);
      ptx::tma_load_2d(base + L::V + kHalf, &tm_kv, kv_full, qcol + 2 * HD + 64, kvrow);
      for (int t = 0; t < n; ++t) {
        const int q = t % kQSlots;
        const int qr = row0 + (i0 + t) * BQ2;
        ptx::mbar_wait(q_empty(q), ((t / kQSlots) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(q_full(q), 2 * kQ2 + 2 * BQ2 * 4);
        const uint32_t sq_ = base + L::Q + q * kQ2, sdo = base + L::dO + q * kQ2;
        ptx::tma_load_2d(sq_, &tm_q, q_full(q), qcol, qr);
        ptx::tma_load_2d(sq_ + kBox64, &tm_q, q_full(q), qcol + 64, qr);
        ptx::tma_load_2d(sdo, &tm_do, q_full(q), head * HD, qr);
        ptx::tma_load_2d(sdo + kBox64, &tm_do, q_full(q), head * HD + 64, qr);
        const int64_t lo = static_cast<int64_t>(head) * p.T + qr;
        ptx::bulk_load_1d(base + L::LD + q * BQ2 * 4, p.lse + lo, BQ2 * 4, q_full(q));
        ptx::bulk_load_1d(base + L::LD + (kQSlots + q) * BQ2 * 4, p.D + lo, BQ2 * 4, q_full(q));
      }
      for (int t = n; t < n + kQSlots; ++t)  // tail: every slot released (each phase waited)
        ptx::mbar_wait(q_empty(t % kQSlots), ((t / kQSlots) & 1) ^ 1);
    }
  } else if (warp == 1) {
    {  // the whole warp runs the issue loop; each tcgen05 op is issued by one elected lane
      constexpr uint32_t id_st = ptx::idesc_bf16_f32(128, BQ2, 0, 0);  // S^T, dP^T: both K-major
      constexpr uint32_t id_kv = ptx::idesc_bf16_f32(128, 128, 0, 1);  // dV, dK (A in TMEM): B MN-major
      constexpr uint32_t id_dq = ptx::idesc_bf16_f32(128, BQ2, 1, 1);  // dQ^T: both MN-major
      // Descriptors built once; per K step only the 14-bit start address moves
      // (a 64-bit add of a compile-time offset >> 4): the single issuing thread
      // must keep up with N=64 MMAs of 32 cycles each.
      auto adv = [](uint64_t d, uint32_t bytes) { return d + (bytes >> 4); };
      const uint64_t k_kmaj = ptx::smem_desc_sw128(base + L::K, 16, 1024);
      const uint64_t v_kmaj = ptx::smem_desc_sw128(base + L::V, 16, 1024);
      const uint64_t k_mnmaj = ptx::smem_desc_sw128(base + L::K, kHalf, 1024);
      auto issue_sdp = [&](int t) {
        const int s = t & 1, q = t % kQSlots;
        ptx::mbar_wait(q_full(q), (t / kQSlots) & 1);
        if (t >= 2) ptx::mbar_wait(s_free(s), ((t - 2) >> 1) & 1);  // dQ^T of block t-2 read out of dP^T[s]
        ptx::tc_fence_after();
        const uint64_t q_kmaj = ptx::smem_desc_sw128(base + L::Q + q * kQ2, 16, 1024);
        const uint64_t do_kmaj = ptx::smem_desc_sw128(base + L::dO + q * kQ2, 16, 1024);
        // S^T[s] overwrites P^T of block t-2: in issue order after dV(t-2), which read it
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          ptx::mma_bf16_ss_w(tS(s), adv(k_kmaj, (kk >> 2) * kHalf + (kk & 3) * 32),
                           adv(q_kmaj, (kk >> 2) * kBox64 + (kk & 3) * 32), id_st, kk > 0 ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          ptx::mma_bf16_ss_w(tdP(s), adv(v_kmaj, (kk >> 2) * kHalf + (kk & 3) * 32),
                           adv(do_kmaj, (kk >> 2) * kBox64 + (kk & 3) * 32), id_st, kk > 0 ? 1u : 0u);
        ptx::mma_commit_w(s_full(s));
      };
      ptx::mbar_wait(kv_full, 0);
      if (n > 0) issue_sdp(0);
      for (int t = 0; t < n; ++t) {
        const int s = t & 1, q = t % kQSlots;
        if (t + 1 < n) issue_sdp(t + 1);  // the next block's products run during this block's softmax
        ptx::mbar_wait(ds_full(s), (t >> 1) & 1);
        ptx::tc_fence_after();
        const uint64_t q_mnmaj = ptx::smem_desc_sw128(base + L::Q + q * kQ2, kBox64, 1024);
        const uint64_t do_mnmaj = ptx::smem_desc_sw128(base + L::dO + q * kQ2, kBox64, 1024);
        const uint64_t ds_mnmaj = ptx::smem_desc_sw128(base + L::dS + s * kPS, kPS, 1024);
#pragma unroll
        for (int kk = 0; kk < BQ2 / 16; ++kk)  // dV += P^T dO  (P^T from TMEM: q 0-31 at cols 0-15, 32-63 at 32-47)
          ptx::mma_bf16_ts_w(tdV, tS(s) + (kk < 2 ? 8 * kk : 32 + 8 * (kk - 2)), adv(do_mnmaj, kk * 2048), id_kv,
                           (t | kk) != 0 ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < BQ2 / 16; ++kk)  // dK += dS^T Q  (dS^T from TMEM, same column layout as P^T)
          ptx::mma_bf16_ts_w(tdK, tdP(s) + (kk < 2 ? 8 * kk : 32 + 8 * (kk - 2)), adv(q_mnmaj, kk * 2048), id_kv,
                           (t | kk) != 0 ? 1u : 0u);
        ptx::mma_commit_w(q_empty(q));  // Q_i, dO_i (and lse, D) no longer read
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk)  // dQ^T = K^T dS^T  (into dP^T[s]: issued after dK, which read dS^T there)
          ptx::mma_bf16_ss_w(tdP(s), adv(k_mnmaj, kk * 2048), adv(ds_mnmaj, kk * 2048), id_dq, kk > 0 ? 1u : 0u);
        ptx::mma_commit_w(dq_full(s));
        ptx::mma_commit_w(p_free(s));  // dS^T smem of block t may be overwritten
      }
      ptx::mma_commit_w(done);
      for (int t = n; t < n + 2; ++t)  // tail: the last dQ^T read-outs (each phase waited)
        if (t >= 2) ptx::mbar_wait(s_free(t & 1), ((t - 2) >> 1) & 1);
    }
  } else if (warp < 10) {
    // ---- softmax warps: lane = key row, 32 query columns each
    const int half = (warp - 2) / 4, q4 = warp % 4;
    const int r = q4 * 32 + lane, c0 = 32 * half;
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const int key = jb * BKV + r;  // position in the sequence
    for (int t = 0; t < n; ++t) {
      const int s = t & 1, q = t % kQSlots, i = i0 + t;
      ptx::mbar_wait(q_full(q), (t / kQSlots) & 1);  // lse, D of the block visible
      ptx::mbar_wait(s_full(s), (t >> 1) & 1);
      ptx::tc_fence_after();
      uint32_t su[32], du[32];
      ptx::tmem_ld_32x32b_x32(tS(s) + lane_off + c0, su);
      ptx::tmem_ld_32x32b_x32(tdP(s) + lane_off + c0, du);
      ptx::tmem_wait_ld();
      if (t >= 2) ptx::mbar_wait(p_free(s), ((t - 2) >> 1) & 1);  // block t-2's MMAs done with sdS[s]
      const float* lse_s = lds + q * BQ2;
      const float* D_s = lds + (kQSlots + q) * BQ2;
      const int qpos0 = i * BQ2 + c0;  // query position of column c0
      const bool need_mask = p.causal && qpos0 < key;  // some column of this thread is masked (q < key)
      uint32_t pk[16], dk[16];
      // pairs of query columns on paired fp32 ops (FMUL2 / FFMA2 / FSUB2)
      const uint64_t sc2 = f2pack(p.scale_log2, p.scale_log2);
      const uint64_t nlog2e = f2pack(-1.4426950408889634f, -1.4426950408889634f);
#pragma unroll
      for (int k = 0; k < 32; k += 2) {
        const float2 l2 = *reinterpret_cast<const float2*>(lse_s + c0 + k);
        const float2 d2 = *reinterpret_cast<const float2*>(D_s + c0 + k);
        float x0, x1;
        f2unpack(ffma2(f2pack(__uint_as_float(su[k]), __uint_as_float(su[k + 1])), sc2,
                       fmul2(f2pack(l2.x, l2.y), nlog2e)),
                 x0, x1);
        float pv[2] = {ex2(x0), ex2(x1)};
#pragma unroll
        for (int u = 0; u < 2; ++u)
          if (need_mask && qpos0 + k + u < key) pv[u] = 0.f;
        const uint64_t pp = f2pack(pv[0], pv[1]);
        float ds0, ds1;
        f2unpack(fmul2(pp, fsub2(f2pack(__uint_as_float(du[k]), __uint_as_float(du[k + 1])), f2pack(d2.x, d2.y))), ds0,
                 ds1);
        pk[k / 2] = pack_bf16(pv[0], pv[1]);
        dk[k / 2] = pack_bf16(ds0, ds1);
      }
      ptx::tmem_st_32x32b_x16(tS(s) + lane_off + c0, pk);   // P^T over this thread's own S^T columns
      ptx::tmem_st_32x32b_x16(tdP(s) + lane_off + c0, dk);  // dS^T over its own dP^T columns (A of dK)
      const uint32_t sds = base + L::dS + s * kPS;
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int c16 = c0 / 8 + v;
        const uint32_t off = static_cast<uint32_t>(r * 128 + ((c16 ^ (r & 7)) << 4));
        st_shared_v4(sds + off, dk[4 * v], dk[4 * v + 1], dk[4 * v + 2], dk[4 * v + 3]);
      }
      ptx::tmem_wait_st();
      ptx::fence_proxy_async();
      ptx::tc_fence_before();
      ptx::mbar_arrive(ds_full(s));
    }
    for (int t = n; t < n + 2; ++t)  // tail: the last dS^T buffers released (each phase waited)
      if (t >= 2) ptx::mbar_wait(p_free(t & 1), ((t - 2) >> 1) & 1);
    // ---- dK (scaled), dV -> dqkv rows of this key block (TMEM lane = key row), 64 columns per thread
    ptx::mbar_wait(done, 0);
    ptx::tc_fence_after();
    const int cc = 64 * half;
    __nv_bfloat16* drow = p.dqkv + static_cast<int64_t>(kvrow + r) * p.ld_dqkv + qcol;
#pragma unroll
    for (int which = 0; which < 2; ++which) {  // 0: dK, 1: dV
      const float f = which == 0 ? p.scale : 1.f;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t u[32];
        ptx::tmem_ld_32x32b_x32((which == 0 ? tdK : tdV) + lane_off + cc + 32 * c, u);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(u[8 * v + 0]) * f, __uint_as_float(u[8 * v + 1]) * f);
          w.y = pack_bf16(__uint_as_float(u[8 * v + 2]) * f, __uint_as_float(u[8 * v + 3]) * f);
          w.z = pack_bf16(__uint_as_float(u[8 * v + 4]) * f, __uint_as_float(u[8 * v + 5]) * f);
          w.w = pack_bf16(__uint_as_float(u[8 * v + 6]) * f, __uint_as_float(u[8 * v + 7]) * f);
          *reinterpret_cast<uint4*>(drow + (which == 0 ? HD : 2 * HD) + cc + 32 * c + 8 * v) = w;
        }
      }
    }
  } else {
    // ---- dQ warps: lane = head-dim row d (quadrant w%4); stage dQ_i [64 q][32 d] fp32, TMA reduce-add
    const int q4 = warp % 4;
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const uint32_t box = base + L::dQ + static_cast<uint32_t>(q4) * kDqBox;
    for (int t = 0; t < n; ++t) {
      const int s = t & 1, i = i0 + t;
      ptx::mbar_wait(dq_full(s), (t >> 1) & 1);
      ptx::tc_fence_after();
      uint32_t qa[32], qb[32];
      ptx::tmem_ld_32x32b_x32(tdP(s) + lane_off, qa);
      ptx::tmem_ld_32x32b_x32(tdP(s) + lane_off + 32, qb);
      ptx::tmem_wait_ld();
      ptx::tc_fence_before();
      ptx::mbar_arrive(s_free(s));  // dP^T[s] may take block t+2's products
      if (lane == 0) ptx::bulk_wait_read0();  // the previous reduce-add has read the staging box
      __syncwarp();
      // element (q, d = lane) of a [64 q][32 d] fp32 SW128 box: row q = 128 B, 16-B chunk (lane / 4) ^ (q & 7)
#pragma unroll
      for (int q = 0; q < 64; ++q) {
        const uint32_t addr = box + q * 128 + ((((lane >> 2) ^ (q & 7)) & 7) << 4) + (lane & 3) * 4;
        const uint32_t val = q < 32 ? qa[q] : qb[q - 32];
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(val) : "memory");
      }
      ptx::fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        ptx::tma_reduce_add_2d(&tm_dq, box, head * HD + 32 * q4, row0 + i * BQ2);
        ptx::bulk_commit();
      }
    }
    if (lane == 0) ptx::bulk_wait0();  // reductions complete before the dQ finalize kernel
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------- backward v3
// v2 made persistent with cluster launch control (as forward v4): the grid is
// one CTA per (key block, head, sequence), but a running CTA takes over
// not-yet-launched CTAs instead of exiting.  Per SM, barrier init and TMEM
// allocation happen once; the next item's K / V load as soon as the current
// item's last MMA has read them, and its first S^T / dP^T products run while
// the softmax warps drain the current item's dK / dV (the first dV / dK MMA of
// an item waits for that drain: acc_free).  Every ring (Q / dO slots, S^T /
// dP^T / dS^T buffers) runs on one block counter across items.
__device__ __forceinline__ void bwd_item(const BwdParams& p, int b, int& jb, int& head, int& row0, int& i0, int& n) {
  const int nseq = p.T / p.seq, per = p.heads * nseq, nkb = p.seq / BKV;
  int rest;
  cta_order(p.grouped, per, nkb, jb, rest, b);
  head = rest % p.heads;
  row0 = (rest / p.heads) * p.seq;
  const int nqb = p.seq / BQ2;
  i0 = p.causal ? 2 * jb : 0;
  n = nqb - i0;
}

__global__ void __launch_bounds__(448, 1) attn_bwd3_kernel(const __grid_constant__ CUtensorMap tm_kv,
                                                           const __grid_constant__ CUtensorMap tm_q,
                                                           const __grid_constant__ CUtensorMap tm_do,
                                                           const __grid_constant__ CUtensorMap tm_dq, BwdParams p) {
  using L = Bwd2Smem;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const float* lds = reinterpret_cast<const float*>(smem_raw + (base - raw) + L::LD);  // lse[3][64], D[3][64]
  const uint32_t bars = base + L::Bars;
  const uint32_t kv_full = bars;
  auto q_full = [&](int q) { return bars + 8 + 8 * q; };    // [3]
  auto q_empty = [&](int q) { return bars + 32 + 8 * q; };  // [3]
  auto s_full = [&](int s) { return bars + 56 + 8 * s; };
  auto ds_full = [&](int s) { return bars + 72 + 8 * s; };
  auto p_free = [&](int s) { return bars + 88 + 8 * s; };
  auto dq_full = [&](int s) { return bars + 104 + 8 * s; };
  auto s_free = [&](int s) { return bars + 120 + 8 * s; };
  const uint32_t done = bars + 136;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw + (bars + 144 - raw));
  const uint32_t kv_empty = bars + 152, acc_free = bars + 160;
  auto clc_full = [&](int s) { return bars + 168 + 8 * s; };
  auto clc_empty = [&](int s) { return bars + 184 + 8 * s; };
  auto clc_resp = [&](int s) { return bars + 208 + 16 * s; };

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    ptx::mbar_init(kv_full, 1);
    ptx::mbar_init(kv_empty, 1);
    ptx::mbar_init(acc_free, 256);
    for (int q = 0; q < kQSlots; ++q) {
      ptx::mbar_init(q_full(q), 1);
      ptx::mbar_init(q_empty(q), 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(s_full(s), 1);
      ptx::mbar_init(ds_full(s), 256);
      ptx::mbar_init(p_free(s), 1);
      ptx::mbar_init(dq_full(s), 1);
      ptx::mbar_init(s_free(s), 128);
      ptx::mbar_init(clc_full(s), 1);
      ptx::mbar_init(clc_empty(s), 13);  // MMA warp, 8 softmax warps, 4 dQ warps
    }
    ptx::mbar_init(done, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc(ptx::smem_u32(tmem_slot), 512);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);
  auto tS = [&](int s) { return tmem + 64u * s; };
  auto tdP = [&](int s) { return tmem + 128u + 64u * s; };
  const uint32_t tdV = tmem + 256, tdK = tmem + 384;
  // successor item (every consumer role; the producer requested it)
  auto next_item = [&](int it) {
    ptx::mbar_wait(clc_full(it & 1), (it >> 1) & 1);
    const int b = clc_next(clc_resp(it & 1));
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(clc_empty(it & 1));
    return b;
  };

  if (warp == 0) {
    if (lane == 0) {
      ptx::prefetch_tmap(&tm_kv);
      ptx::prefetch_tmap(&tm_q);
      ptx::prefetch_tmap(&tm_do);
      int g = 0;
      for (int b = static_cast<int>(blockIdx.x), it = 0; b >= 0; ++it) {
        int jb, head, row0, i0, n;
        bwd_item(p, b, jb, head, row0, i0, n);
        const int qcol = head * 3 * HD, kvrow = row0 + jb * BKV;
        ptx::mbar_wait(kv_empty, (it & 1) ^ 1);  // the previous item's MMAs are done with K / V
        ptx::mbar_arrive_expect_tx(kv_full, 2 * kTile);
        ptx::tma_load_2d(base + L::K, &tm_kv, kv_full, qcol + HD, kvrow);
        ptx::tma_load_2d(base + L::K + kHalf, &tm_kv, kv_full, qcol + HD + 64, kvrow);
        ptx::tma_load_2d(base + L::V, &tm_kv, kv_full, qcol + 2 * HD, kvrow);
        ptx::tma_load_2d(base + L::V + kHalf, &tm_kv, kv_full, qcol + 2 * HD + 64, kvrow);
        for (int t = 0; t < n; ++t, ++g) {
          const int q = g % kQSlots;
          const int qr = row0 + (i0 + t) * BQ2;
          ptx::mbar_wait(q_empty(q), ((g / kQSlots) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(q_full(q), 2 * kQ2 + 2 * BQ2 * 4);
          const uint32_t sq_ = base + L::Q + q * kQ2, sdo = base + L::dO + q * kQ2;
          ptx::tma_load_2d(sq_, &tm_q, q_full(q), qcol, qr);
          ptx::tma_load_2d(sq_ + kBox64, &tm_q, q_full(q), qcol + 64, qr);
          ptx::tma_load_2d(sdo, &tm_do, q_full(q), head * HD, qr);
          ptx::tma_load_2d(sdo + kBox64, &tm_do, q_full(q), head * HD + 64, qr);
          const int64_t lo = static_cast<int64_t>(head) * p.T + qr;
          ptx::bulk_load_1d(base + L::LD + q * BQ2 * 4, p.lse + lo, BQ2 * 4, q_full(q));
          ptx::bulk_load_1d(base + L::LD + (kQSlots + q) * BQ2 * 4, p.D + lo, BQ2 * 4, q_full(q));
          if (t + 1 == n) {  // ask for the successor with the last Q / dO load (as forward v4)
            const int cs = it & 1;
            ptx::mbar_wait(clc_empty(cs), ((it >> 1) & 1) ^ 1);
            ptx::fence_proxy_async();
            ptx::mbar_arrive_expect_tx(clc_full(cs), 16);
            clc_try_cancel(clc_resp(cs), clc_full(cs));
          }
        }
        ptx::mbar_wait(clc_full(it & 1), (it >> 1) & 1);
        b = clc_next(clc_resp(it & 1));
      }
      for (int t = g; t < g + kQSlots; ++t)  // tail: every slot released (each phase waited)
        ptx::mbar_wait(q_empty(t % kQSlots), ((t / kQSlots) & 1) ^ 1);
    }
  } else if (warp == 1) {
    constexpr uint32_t id_st = ptx::idesc_bf16_f32(128, BQ2, 0, 0);
    constexpr uint32_t id_kv = ptx::idesc_bf16_f32(128, 128, 0, 1);
    constexpr uint32_t id_dq = ptx::idesc_bf16_f32(128, BQ2, 1, 1);
    auto adv = [](uint64_t d, uint32_t bytes) { return d + (bytes >> 4); };
    const uint64_t k_kmaj = ptx::smem_desc_sw128(base + L::K, 16, 1024);
    const uint64_t v_kmaj = ptx::smem_desc_sw128(base + L::V, 16, 1024);
    const uint64_t k_mnmaj = ptx::smem_desc_sw128(base + L::K, kHalf, 1024);
    auto issue_sdp = [&](int g) {
      const int s = g & 1, q = g % kQSlots;
      ptx::mbar_wait(q_full(q), (g / kQSlots) & 1);
      if (g >= 2) ptx::mbar_wait(s_free(s), ((g - 2) >> 1) & 1);
      ptx::tc_fence_after();
      const uint64_t q_kmaj = ptx::smem_desc_sw128(base + L::Q + q * kQ2, 16, 1024);
      const uint64_t do_kmaj = ptx::smem_desc_sw128(base + L::dO + q * kQ2, 16, 1024);
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk)
        ptx::mma_bf16_ss_w(tS(s), adv(k_kmaj, (kk >> 2) * kHalf + (kk & 3) * 32),
                           adv(q_kmaj, (kk >> 2) * kBox64 + (kk & 3) * 32), id_st, kk > 0 ? 1u : 0u);
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk)
        ptx::mma_bf16_ss_w(tdP(s), adv(v_kmaj, (kk >> 2) * kHalf + (kk & 3) * 32),
                           adv(do_kmaj, (kk >> 2) * kBox64 + (kk & 3) * 32), id_st, kk > 0 ? 1u : 0u);
      ptx::mma_commit_w(s_full(s));
    };
    int g0 = 0;
    for (int b = static_cast<int>(blockIdx.x), it = 0; b >= 0; ++it) {
      int jb, head, row0, i0, n;
      bwd_item(p, b, jb, head, row0, i0, n);
      ptx::mbar_wait(kv_full, it & 1);
      ptx::tc_fence_after();
      if (n > 0) issue_sdp(g0);
      for (int t = 0; t < n; ++t) {
        const int g = g0 + t, s = g & 1, q = g % kQSlots;
        if (t + 1 < n) issue_sdp(g + 1);
        ptx::mbar_wait(ds_full(s), (g >> 1) & 1);
        if (t == 0) ptx::mbar_wait(acc_free, (it & 1) ^ 1);  // the previous item's dK / dV drained
        ptx::tc_fence_after();
        const uint64_t q_mnmaj = ptx::smem_desc_sw128(base + L::Q + q * kQ2, kBox64, 1024);
        const uint64_t do_mnmaj = ptx::smem_desc_sw128(base + L::dO + q * kQ2, kBox64, 1024);
        const uint64_t ds_mnmaj = ptx::smem_desc_sw128(base + L::dS + s * kPS, kPS, 1024);
#pragma unroll
        for (int kk = 0; kk < BQ2 / 16; ++kk)
          ptx::mma_bf16_ts_w(tdV, tS(s) + (kk < 2 ? 8 * kk : 32 + 8 * (kk - 2)), adv(do_mnmaj, kk * 2048), id_kv,
                             (t | kk) != 0 ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < BQ2 / 16; ++kk)
          ptx::mma_bf16_ts_w(tdK, tdP(s) + (kk < 2 ? 8 * kk : 32 + 8 * (kk - 2)), adv(q_mnmaj, kk * 2048), id_kv,
                             (t | kk) != 0 ? 1u : 0u);
        ptx::mma_commit_w(q_empty(q));
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk)
          ptx::mma_bf16_ss_w(tdP(s), adv(k_mnmaj, kk * 2048), adv(ds_mnmaj, kk * 2048), id_dq, kk > 0 ? 1u : 0u);
        ptx::mma_commit_w(dq_full(s));
        ptx::mma_commit_w(p_free(s));
      }
      ptx::mma_commit_w(done);      // dK / dV of this item complete
      ptx::mma_commit_w(kv_empty);  // K / V no longer read
      g0 += n;
      b = next_item(it);
    }
    for (int t = g0; t < g0 + 2; ++t)  // tail: the last dQ^T read-outs (each phase waited)
      if (t >= 2) ptx::mbar_wait(s_free(t & 1), ((t - 2) >> 1) & 1);
  } else if (warp < 10) {
    const int half = (warp - 2) / 4, q4 = warp % 4;
    const int r = q4 * 32 + lane, c0 = 32 * half;
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    int g = 0;
    for (int b = static_cast<int>(blockIdx.x), it = 0; b >= 0; ++it) {
      int jb, head, row0, i0, n;
      bwd_item(p, b, jb, head, row0, i0, n);
      const int key = jb * BKV + r;
      for (int t = 0; t < n; ++t, ++g) {
        const int s = g & 1, q = g % kQSlots, i = i0 + t;
        ptx::mbar_wait(q_full(q), (g / kQSlots) & 1);
        ptx::mbar_wait(s_full(s), (g >> 1) & 1);
        ptx::tc_fence_after();
        uint32_t su[32], du[32];
        ptx::tmem_ld_32x32b_x32(tS(s) + lane_off + c0, su);
        ptx::tmem_ld_32x32b_x32(tdP(s) + lane_off + c0, du);
        ptx::tmem_wait_ld();
        if (g >= 2) ptx::mbar_wait(p_free(s), ((g - 2) >> 1) & 1);
        const float* lse_s = lds + q * BQ2;
        const float* D_s = lds + (kQSlots + q) * BQ2;
        const int qpos0 = i * BQ2 + c0;
        const bool need_mask = p.causal && qpos0 < key;
        uint32_t pk[16], dk[16];
        const uint64_t sc2 = f2pack(p.scale_log2, p.scale_log2);
        const uint64_t nlog2e = f2pack(-1.4426950408889634f, -1.4426950408889634f);
#pragma unroll
        for (int k = 0; k < 32; k += 2) {
          const float2 l2 = *reinterpret_cast<const float2*>(lse_s + c0 + k);
          const float2 d2 = *reinterpret_cast<const float2*>(D_s + c0 + k);
          float x0, x1;
          f2unpack(ffma2(f2pack(__uint_as_float(su[k]), __uint_as_float(su[k + 1])), sc2,
                         fmul2(f2pack(l2.x, l2.y), nlog2e)),
                   x0, x1);
          float pv[2] = {ex2(x0), ex2(x1)};
#pragma unroll
          for (int u = 0; u < 2; ++u)
            if (need_mask && qpos0 + k + u < key) pv[u] = 0.f;
          const uint64_t pp = f2pack(pv[0], pv[1]);
          float ds0, ds1;
          f2unpack(fmul2(pp, fsub2(f2pack(__uint_as_float(du[k]), __uint_as_float(du[k + 1])), f2pack(d2.x, d2.y))),
                   ds0, ds1);
          pk[k / 2] = pack_bf16(pv[0], pv[1]);
          dk[k / 2] = pack_bf16(ds0, ds1);
        }
        ptx::tmem_st_32x32b_x16(tS(s) + lane_off + c0, pk);
        ptx::tmem_st_32x32b_x16(tdP(s) + lane_off + c0, dk);
        const uint32_t sds = base + L::dS + s * kPS;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int c16 = c0 / 8 + v;
          const uint32_t off = static_cast<uint32_t>(r * 128 + ((c16 ^ (r & 7)) << 4));
          st_shared_v4(sds + off, dk[4 * v], dk[4 * v + 1], dk[4 * v + 2], dk[4 * v + 3]);
        }
        ptx::tmem_wait_st();
        ptx::fence_proxy_async();
        ptx::tc_fence_before();
        ptx::mbar_arrive(ds_full(s));
      }
      // dK (scaled), dV of this item -> dqkv rows of its key block
      ptx::mbar_wait(done, it & 1);
      ptx::tc_fence_after();
      const int cc = 64 * half, kvrow = row0 + jb * BKV;
      __nv_bfloat16* drow = p.dqkv + static_cast<int64_t>(kvrow + r) * p.ld_dqkv + head * 3 * HD;
#pragma unroll
      for (int which = 0; which < 2; ++which) {
        const float f = which == 0 ? p.scale : 1.f;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t u[32];
          ptx::tmem_ld_32x32b_x32((which == 0 ? tdK : tdV) + lane_off + cc + 32 * c, u);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            uint4 w;
            w.x = pack_bf16(__uint_as_float(u[8 * v + 0]) * f, __uint_as_float(u[8 * v + 1]) * f);
            w.y = pack_bf16(__uint_as_float(u[8 * v + 2]) * f, __uint_as_float(u[8 * v + 3]) * f);
            w.z = pack_bf16(__uint_as_float(u[8 * v + 4]) * f, __uint_as_float(u[8 * v + 5]) * f);
            w.w = pack_bf16(__uint_as_float(u[8 * v + 6]) * f, __uint_as_float(u[8 * v + 7]) * f);
            *reinterpret_cast<uint4*>(drow + (which == 0 ? HD : 2 * HD) + cc + 32 * c + 8 * v) = w;
          }
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(acc_free);
      b = next_item(it);
    }
    for (int t = g; t < g + 2; ++t)  // tail: the last dS^T buffers released (each phase waited)
      if (t >= 2) ptx::mbar_wait(p_free(t & 1), ((t - 2) >> 1) & 1);
  } else {
    const int q4 = warp % 4;
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const uint32_t box = base + L::dQ + static_cast<uint32_t>(q4) * kDqBox;
    int g = 0;
    for (int b = static_cast<int>(blockIdx.x), it = 0; b >= 0; ++it) {
      int jb, head, row0, i0, n;
      bwd_item(p, b, jb, head, row0, i0, n);
      for (int t = 0; t < n; ++t, ++g) {
        const int s = g & 1, i = i0 + t;
        ptx::mbar_wait(dq_full(s), (g >> 1) & 1);
        ptx::tc_fence_after();
        uint32_t qa[32], qb[32];
        ptx::tmem_ld_32x32b_x32(tdP(s) + lane_off, qa);
        ptx::tmem_ld_32x32b_x32(tdP(s) + lane_off + 32, qb);
        ptx::tmem_wait_ld();
        ptx::tc_fence_before();
        ptx::mbar_arrive(s_free(s));
        if (lane == 0) ptx::bulk_wait_read0();
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 64; ++q) {
          const uint32_t addr = box + q * 128 + ((((lane >> 2) ^ (q & 7)) & 7) << 4) + (lane & 3) * 4;
          const uint32_t val = q < 32 ? qa[q] : qb[q - 32];
          asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(val) : "memory");
        }
        ptx::fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          ptx::tma_reduce_add_2d(&tm_dq, box, head * HD + 32 * q4, row0 + i * BQ2);
          ptx::bulk_commit();
        }
      }
      b = next_item(it);
    }
    if (lane == 0) ptx::bulk_wait0();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// D[h][t] = sum_c dO[t, h*128 + c] * O[t, h*128 + c] (fp32); zero the dQ accumulator.
// One warp per (row, head).
__global__ void attn_bwd_prep_kernel(const __nv_bfloat16* __restrict__ o, int64_t ld_o,
                                     const __nv_bfloat16* __restrict__ dO, int64_t ld_do, int T, int heads,
                                     float* __restrict__ D, float* __restrict__ dq_acc) {
  const int lane = threadIdx.x % 32;
  const int64_t nw = static_cast<int64_t>(T) * heads;
  for (int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32; w < nw;
       w += (static_cast<int64_t>(gridDim.x) * blockDim.x) / 32) {
    const int t = static_cast<int>(w / heads), h = static_cast<int>(w % heads);
    const uint2 a = *reinterpret_cast<const uint2*>(o + t * ld_o + h * HD + 4 * lane);
    const uint2 b = *reinterpret_cast<const uint2*>(dO + t * ld_do + h * HD + 4 * lane);
    const __nv_bfloat162* ah = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* bh = reinterpret_cast<const __nv_bfloat162*>(&b);
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float2 x = __bfloat1622float2(ah[i]), y = __bfloat1622float2(bh[i]);
      acc += x.x * y.x + x.y * y.y;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) D[static_cast<int64_t>(h) * T + t] = acc;
    *reinterpret_cast<float4*>(dq_acc + static_cast<int64_t>(t) * heads * HD + h * HD + 4 * lane) =
        make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// dqkv[t, 3h*128 + c] = bf16(dq_acc[t, h*128 + c] / sqrt(d)).
__global__ void attn_bwd_dq_kernel(const float* __restrict__ dq_acc, int T, int heads, float scale,
                                   __nv_bfloat16* __restrict__ dqkv, int64_t ld) {
  const int64_t n8 = static_cast<int64_t>(T) * heads * HD / 8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t e = i * 8;
    const int t = static_cast<int>(e / (heads * HD));
    const int rem = static_cast<int>(e % (heads * HD));
    const int h = rem / HD, c = rem % HD;
    const float4 a = *reinterpret_cast<const float4*>(dq_acc + e);
    const float4 b = *reinterpret_cast<const float4*>(dq_acc + e + 4);
    uint4 w;
    w.x = pack_bf16(a.x * scale, a.y * scale);
    w.y = pack_bf16(a.z * scale, a.w * scale);
    w.z = pack_bf16(b.x * scale, b.y * scale);
    w.w = pack_bf16(b.z * scale, b.w * scale);
    *reinterpret_cast<uint4*>(dqkv + t * ld + h * 3 * HD + c) = w;
  }
}

constexpr int kBwdSmem = 6 * kTile + 128 + 1024;

}  // namespace

const char* attn_check(int64_t T, int64_t seq, int heads, int head_dim, int64_t ld_qkv, int64_t ld_ctx) {
  if (head_dim != HD) return "attention: head_dim must be 128";
  if (heads <= 0 || T <= 0 || seq <= 0) return "attention: T, seq, heads must be positive";
  if (seq % BQ) return "attention: seq must be a multiple of 128";
  if (T % seq) return "attention: T must be whole sequences (T % seq == 0)";
  if (ld_qkv < 3 * heads * HD || ld_ctx < heads * HD) return "attention: leading dimension too small";
  if ((ld_qkv % 8) || (ld_ctx % 8)) return "attention: leading dimensions must be multiples of 8 elements";
  if (T > (int64_t(1) << 30)) return "attention: T too large";
  return nullptr;
}

// Split-KV combine: one warp per (query row, head), 4 columns per lane.
__global__ void attn_fwd_combine_kernel(FwdParams p) {
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (w >= static_cast<int64_t>(p.T) * p.heads) return;
  const int64_t row = w / p.heads;
  const int head = static_cast<int>(w % p.heads);
  float mx = -INFINITY;
  for (int s = 0; s < p.kv_split; ++s) mx = fmaxf(mx, p.mlpart[((s * static_cast<int64_t>(p.T) + row) * p.heads + head) * 2]);
  float L = 0.f, o[4] = {0.f, 0.f, 0.f, 0.f};
  for (int s = 0; s < p.kv_split; ++s) {
    const float* ml = p.mlpart + ((s * static_cast<int64_t>(p.T) + row) * p.heads + head) * 2;
    if (ml[1] == 0.f) continue;  // empty share
    const float f = ex2(ml[0] - mx);
    L += f * ml[1];
    const float4 v = reinterpret_cast<const float4*>(p.opart + (s * static_cast<int64_t>(p.T) + row) * (p.heads * HD) +
                                                     head * HD)[lane];
    o[0] += f * v.x;
    o[1] += f * v.y;
    o[2] += f * v.z;
    o[3] += f * v.w;
  }
  const float inv = 1.f / L;
  uint2 pk;
  pk.x = pack_bf16(o[0] * inv, o[1] * inv);
  pk.y = pack_bf16(o[2] * inv, o[3] * inv);
  *reinterpret_cast<uint2*>(p.ctx + row * p.ld_ctx + head * HD + 4 * lane) = pk;
  if (lane == 0) p.lse[static_cast<int64_t>(head) * p.T + row] = (mx + log2f(L)) * kLn2;
}

// KV splits of the forward v2 on this shape: enough CTAs for one wave when
// the (sequence, head, query-tile pair) grid is smaller than the GPU (chunked
// layers at N > 1: e.g. 40 CTAs), at most 4 and at most the KV blocks.
int attn_fwd_splits(int64_t T, int64_t seq, int heads) {
  const int64_t grid = ((seq / BQ + 1) / 2) * heads * (T / seq);
  if (grid <= 0 || grid >= num_sms()) return 1;
  int s = static_cast<int>((num_sms() + grid - 1) / grid);
  s = min(s, 4);
  s = min(s, static_cast<int>(seq / BKV));
  return s < 1 ? 1 : s;
}

size_t attn_fwd_split_bytes(int64_t T, int64_t seq, int heads) {
  const int s = attn_fwd_splits(T, seq, heads);
  return s > 1 ? static_cast<size_t>(s) * T * heads * (HD + 2) * 4 : 0;
}

cudaError_t attn_fwd_launch(const void* qkv, int64_t ld_qkv, int T, int seq, int heads, int causal, void* ctx,
                            int64_t ld_ctx, float* lse, cudaStream_t st, void* ws, size_t ws_bytes) {
  alignas(64) CUtensorMap tm;
  if (!tmap_bf16_2d(&tm, qkv, T, 3 * heads * HD, ld_qkv, 128, 64)) return cudaErrorInvalidValue;
  // ATP_ATTN_FWD = 1 / 2 / 3 / 4: forward kernel version (default 4, v2 made
  // persistent with cluster launch control: b4 s2048 32 heads causal 0.167 ->
  // 0.152 ms, 40 heads 0.215 -> 0.193, non-causal 0.257 -> 0.250, s8192 0.120
  // -> 0.123: profiles/r02_attn_persistent.log; v3, two softmax threads per
  // row, measured 4-5% slower than v2: profiles/r02_attn_fwd_v3.log).  Grids
  // smaller than the GPU take v2 with split-KV.
  static const int fwd_ver = [] {
    const char* e = getenv("ATP_ATTN_FWD");
    return e ? atoi(e) : 4;
  }();
  const bool v1 = fwd_ver == 1;
  static bool attr = [] {
    return cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFwdSmem) ==
               cudaSuccess &&
           cudaFuncSetAttribute(attn_fwd2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFwdSmem) ==
               cudaSuccess &&
           cudaFuncSetAttribute(attn_fwd3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFwd3Smem) ==
               cudaSuccess &&
           cudaFuncSetAttribute(attn_fwd4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFwd4Smem) ==
               cudaSuccess;
  }();
  (void)attr;
  static const bool grouped = [] {
    const char* e = getenv("ATP_ATTN_ORDER");
    return !(e && e[0] == '0');
  }();
  FwdParams p;
  {
    // chunks of up to one wave of CTAs (the K/V of G (sequence, head) groups stay
    // in L2 while their query-tile pairs stream them), heaviest first inside a
    // chunk: b4 s2048 32 heads causal 0.178 -> 0.167 ms, 40 heads 0.238 -> 0.217,
    // non-causal 0.304 -> 0.261 ms (sweep: profiles/r01_attn_fwd_order.log)
    const int per_group = (seq / BQ + 1) / 2;  // CTAs of one (sequence, head): query-tile pairs
    static const int g_env = [] {  // A/B: ATP_ATTN_FWD_G = groups per chunk
      const char* e = getenv("ATP_ATTN_FWD_G");
      return e ? atoi(e) : -1;
    }();
    // G = the largest power of two with G * per_group <= SMs (16 at s = 2048):
    // measured best of G in {0, 8, 12, 14, 16, 18, 37, 74, 128} on both head
    // counts; for long sequences (per_group > 16) the in-chunk causal imbalance
    // costs more than the reuse gains, so global heaviest-first order
    int G = 0;
    if (per_group <= 16)
      for (G = 1; 2 * G * per_group <= num_sms(); G *= 2) {
      }
    p.grouped = !grouped ? 0 : g_env >= 0 ? g_env : G;
  }
  p.T = T;
  p.seq = seq;
  p.heads = heads;
  p.causal = causal ? 1 : 0;
  p.scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(HD));
  p.ctx = static_cast<__nv_bfloat16*>(ctx);
  p.ld_ctx = ld_ctx;
  p.lse = lse;
  if (v1) {
    attn_fwd_kernel<<<(seq / BQ) * heads * (T / seq), 256, kFwdSmem, st>>>(tm, p);
  } else if (fwd_ver == 2 || fwd_ver == 4) {
    // split-KV when the grid is smaller than the GPU and the caller gave the workspace
    static const bool split_on = [] {
      const char* e = getenv("ATP_ATTN_SPLIT");
      return !(e && e[0] == '0');
    }();
    const int S = split_on ? attn_fwd_splits(T, seq, heads) : 1;
    if (S > 1 && ws != nullptr && ws_bytes >= attn_fwd_split_bytes(T, seq, heads)) {
      p.kv_split = S;
      p.opart = static_cast<float*>(ws);
      p.mlpart = p.opart + static_cast<size_t>(S) * T * heads * HD;
      attn_fwd2_kernel<<<((seq / BQ + 1) / 2) * heads * (T / seq) * S, 320, kFwdSmem, st>>>(tm, p);
      const int64_t warps = static_cast<int64_t>(T) * heads;
      attn_fwd_combine_kernel<<<static_cast<unsigned>((warps * 32 + 255) / 256), 256, 0, st>>>(p);
    } else if (fwd_ver == 4 && p.grouped > 0) {
      // persistent for the chunked (grouped) CTA order, seq <= 4096; longer
      // sequences (global heaviest-first order, items of 30+ steps) keep v2:
      // b1 s8192 0.120 (v2) vs 0.123 ms (v4), profiles/r02_attn_persistent.log
      attn_fwd4_kernel<<<((seq / BQ + 1) / 2) * heads * (T / seq), 320, kFwd4Smem, st>>>(tm, p);
    } else {
      attn_fwd2_kernel<<<((seq / BQ + 1) / 2) * heads * (T / seq), 320, kFwdSmem, st>>>(tm, p);
    }
  } else {
    attn_fwd3_kernel<<<((seq / BQ + 1) / 2) * heads * (T / seq), kFwd3Threads, kFwd3Smem, st>>>(tm, p);
  }
  return cudaGetLastError();
}

size_t attn_workspace_bytes(int64_t T, int heads) {
  return static_cast<size_t>(T) * heads * HD * 4 + static_cast<size_t>(T) * heads * 4;
}

cudaError_t attn_bwd_launch(const void* qkv, int64_t ld_qkv, const void* ctx, int64_t ld_ctx, const float* lse,
                            const void* dctx, int64_t ld_dctx, int T, int seq, int heads, int causal, void* dqkv,
                            int64_t ld_dqkv, void* workspace, cudaStream_t st) {
  alignas(64) CUtensorMap tq, td, tdq;
  if (!tmap_bf16_2d(&tq, qkv, T, 3 * heads * HD, ld_qkv, 128, 64)) return cudaErrorInvalidValue;
  if (!tmap_bf16_2d(&td, dctx, T, heads * HD, ld_dctx, 128, 64)) return cudaErrorInvalidValue;
  if (!tmap_f32_2d(&tdq, workspace, T, heads * HD, heads * HD, 128, 32)) return cudaErrorInvalidValue;
  static bool attr = [] {
    return cudaFuncSetAttribute(attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kBwdSmem) ==
           cudaSuccess;
  }();
  (void)attr;
  float* dq_acc = static_cast<float*>(workspace);
  float* D = dq_acc + static_cast<int64_t>(T) * heads * HD;
  const int sms = num_sms();
  attn_bwd_prep_kernel<<<sms * 8, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(ctx), ld_ctx,
                                                static_cast<const __nv_bfloat16*>(dctx), ld_dctx, T, heads, D, dq_acc);
  static const bool grouped = [] {
    const char* e = getenv("ATP_ATTN_ORDER");
    return !(e && e[0] == '0');
  }();
  BwdParams p;
  // chunks of G (sequence, head) groups of seq/128 key-block CTAs each, so the
  // Q / dO / lse / D blocks of a chunk stay in L2: seq <= 2048, the largest power
  // of two with G * CTAs-per-group <= SMs (like the forward); longer sequences
  // ~4 waves of CTAs.  Sweep (G = 8..128, b4 s2048 / b1 s8192): G in 8..37 within
  // 1% causal, G = 8 best non-causal (0.787 vs 0.811 ms at G = 37), 64+ worse.
  static const int gb_env = [] {  // A/B: ATP_ATTN_BWD_G = groups per chunk
    const char* e = getenv("ATP_ATTN_BWD_G");
    return e ? atoi(e) : -1;
  }();
  {
    const int per_group = seq / BKV;
    int G = 0;
    if (per_group <= 16) {
      for (G = 1; 2 * G * per_group <= num_sms(); G *= 2) {
      }
    } else {
      G = (4 * num_sms() + per_group - 1) / per_group;
    }
    p.grouped = !grouped ? 0 : gb_env >= 0 ? gb_env : G;
  }
  p.T = T;
  p.seq = seq;
  p.heads = heads;
  p.causal = causal ? 1 : 0;
  p.scale = 1.f / sqrtf(static_cast<float>(HD));
  p.scale_log2 = 1.4426950408889634f * p.scale;
  p.lse = lse;
  p.D = D;
  p.dq_acc = dq_acc;
  p.dqkv = static_cast<__nv_bfloat16*>(dqkv);
  p.ld_dqkv = ld_dqkv;
  const int grid = (seq / BKV) * heads * (T / seq);
  // ATP_ATTN_BWD = 1 / 2 / 3: backward kernel version (default 3, v2 made
  // persistent with cluster launch control: b4 s2048 32 heads causal 0.498 ->
  // 0.470 ms, non-causal 0.776 -> 0.757: profiles/r02_attn_persistent.log)
  static const int bwd_ver = [] {
    const char* e = getenv("ATP_ATTN_BWD");
    return e ? atoi(e) : 3;
  }();
  if (bwd_ver == 1) {
    attn_bwd_kernel<<<grid, 320, kBwdSmem, st>>>(tq, td, tdq, p);
  } else {
    alignas(64) CUtensorMap tq64, td64, tdq64;
    if (!tmap_bf16_2d(&tq64, qkv, T, 3 * heads * HD, ld_qkv, BQ2, 64)) return cudaErrorInvalidValue;
    if (!tmap_bf16_2d(&td64, dctx, T, heads * HD, ld_dctx, BQ2, 64)) return cudaErrorInvalidValue;
    if (!tmap_f32_2d(&tdq64, workspace, T, heads * HD, heads * HD, BQ2, 32)) return cudaErrorInvalidValue;
    static bool attr2 = cudaFuncSetAttribute(attn_bwd2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             Bwd2Smem::Bytes) == cudaSuccess;
    (void)attr2;
    if (bwd_ver == 3) {
      static bool attr3 = cudaFuncSetAttribute(attn_bwd3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               Bwd2Smem::Bytes) == cudaSuccess;
      (void)attr3;
      attn_bwd3_kernel<<<grid, 448, Bwd2Smem::Bytes, st>>>(tq, tq64, td64, tdq64, p);
    } else {
      attn_bwd2_kernel<<<grid, 448, Bwd2Smem::Bytes, st>>>(tq, tq64, td64, tdq64, p);
    }
  }
  attn_bwd_dq_kernel<<<sms * 8, 256, 0, st>>>(dq_acc, T, heads, p.scale, static_cast<__nv_bfloat16*>(dqkv), ld_dqkv);
  return cudaGetLastError();
}

}  // namespace atp
