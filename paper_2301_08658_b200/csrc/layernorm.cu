// Full-layer memory-bound kernels: LayerNorm with the
// hidden dimension sharded over mesh dim 2 (reading G33), and the block
// pack / unpack around the dim-2 reduce-scatter / all-gather of the attention
// heads (Fig. 6(a); reading G32).
//
// LayerNorm rows are split in two passes around a [rows, 2] fp32 all-reduce:
//   ln_stats        s = (sum x, sum x^2) over the local columns
//   ln_apply        mean = s0/n, rstd = 1/sqrt(s1/n - mean^2 + eps);
//                   y = (x - mean) * rstd * gamma + beta; saves (mean, rstd)
//   ln_bwd_stats    s = (sum g, sum g*xhat), g = dy * gamma
//   ln_bwd_apply    out = res + rstd * (g - s0/n - xhat * s1/n)
//   ln_param_grad   dgamma = sum_rows dy*xhat, dbeta = sum_rows dy (fp32,
//                   deterministic: fixed row segments, then a fixed-order sum)
// One warp per row, 16-byte vectors; grids are multiples of the SM count.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "atp_internal.h"
#include "elementwise.h"

namespace atp {

namespace {

constexpr float kLnEps = 1e-5f;  // reading G29 (Megatron / PyTorch default)
constexpr int kSegs = 128;       // row segments of ln_param_grad (x cols/2048 CTAs)

struct F8 {
  float v[8];
};
__device__ __forceinline__ F8 ld8(const __nv_bfloat16* p) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
  F8 r;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    r.v[2 * i] = f.x;
    r.v[2 * i + 1] = f.y;
  }
  return r;
}
__device__ __forceinline__ void st8(__nv_bfloat16* p, const F8& f) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f.v[2 * i], f.v[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

int grid_for(int64_t warps_needed) {
  const int64_t blocks = (warps_needed + 7) / 8;
  const int64_t cap = static_cast<int64_t>(num_sms()) * 8;
  return static_cast<int>(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

__global__ void ln_stats_kernel(const __nv_bfloat16* __restrict__ x, int64_t ldx, int64_t rows, int64_t cols,
                                float* __restrict__ out) {
  const int lane = threadIdx.x % 32;
  for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32; r < rows;
       r += (static_cast<int64_t>(gridDim.x) * blockDim.x) / 32) {
    float s = 0.f, q = 0.f;
    for (int64_t c = 8 * lane; c < cols; c += 256) {
      const F8 v = ld8(x + r * ldx + c);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        s += v.v[i];
        q += v.v[i] * v.v[i];
      }
    }
    s = warp_sum(s);
    q = warp_sum(q);
    if (lane == 0) {
      out[2 * r] = s;
      out[2 * r + 1] = q;
    }
  }
}

__global__ void ln_apply_kernel(const __nv_bfloat16* __restrict__ x, int64_t ldx, int64_t rows, int64_t cols,
                                const float* __restrict__ stats, float n_total, const __nv_bfloat16* __restrict__ gamma,
                                const __nv_bfloat16* __restrict__ beta, __nv_bfloat16* __restrict__ y, int64_t ldy,
                                float* __restrict__ saved) {
  const int lane = threadIdx.x % 32;
  for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32; r < rows;
       r += (static_cast<int64_t>(gridDim.x) * blockDim.x) / 32) {
    const float mean = stats[2 * r] / n_total;
    const float var = fmaxf(stats[2 * r + 1] / n_total - mean * mean, 0.f);
    const float rstd = rsqrtf(var + kLnEps);
    for (int64_t c = 8 * lane; c < cols; c += 256) {
      const F8 v = ld8(x + r * ldx + c), g = ld8(gamma + c), b = ld8(beta + c);
      F8 o;
#pragma unroll
      for (int i = 0; i < 8; ++i) o.v[i] = (v.v[i] - mean) * rstd * g.v[i] + b.v[i];
      st8(y + r * ldy + c, o);
    }
    if (lane == 0) {
      saved[2 * r] = mean;
      saved[2 * r + 1] = rstd;
    }
  }
}

__global__ void ln_bwd_stats_kernel(const __nv_bfloat16* __restrict__ dy, int64_t lddy, const __nv_bfloat16* __restrict__ x,
                                    int64_t ldx, int64_t rows, int64_t cols, const __nv_bfloat16* __restrict__ gamma,
                                    const float* __restrict__ saved, float* __restrict__ out) {
  const int lane = threadIdx.x % 32;
  for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32; r < rows;
       r += (static_cast<int64_t>(gridDim.x) * blockDim.x) / 32) {
    const float mean = saved[2 * r], rstd = saved[2 * r + 1];
    float s = 0.f, q = 0.f;
    for (int64_t c = 8 * lane; c < cols; c += 256) {
      const F8 d = ld8(dy + r * lddy + c), v = ld8(x + r * ldx + c), g = ld8(gamma + c);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float gg = d.v[i] * g.v[i];
        s += gg;
        q += gg * (v.v[i] - mean) * rstd;
      }
    }
    s = warp_sum(s);
    q = warp_sum(q);
    if (lane == 0) {
      out[2 * r] = s;
      out[2 * r + 1] = q;
    }
  }
}

__global__ void ln_bwd_apply_kernel(const __nv_bfloat16* __restrict__ dy, int64_t lddy, const __nv_bfloat16* __restrict__ x,
                                    int64_t ldx, int64_t rows, int64_t cols, const __nv_bfloat16* __restrict__ gamma,
                                    const float* __restrict__ saved, const float* __restrict__ sums, float n_total,
                                    const __nv_bfloat16* res, int64_t ldres, __nv_bfloat16* out, int64_t ldo) {
  const int lane = threadIdx.x % 32;
  for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32; r < rows;
       r += (static_cast<int64_t>(gridDim.x) * blockDim.x) / 32) {
    const float mean = saved[2 * r], rstd = saved[2 * r + 1];
    const float m1 = sums[2 * r] / n_total, m2 = sums[2 * r + 1] / n_total;
    for (int64_t c = 8 * lane; c < cols; c += 256) {
      const F8 d = ld8(dy + r * lddy + c), v = ld8(x + r * ldx + c), g = ld8(gamma + c);
      const F8 rr = ld8(res + r * ldres + c);
      F8 o;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float xh = (v.v[i] - mean) * rstd;
        o.v[i] = rr.v[i] + rstd * (d.v[i] * g.v[i] - m1 - xh * m2);
      }
      st8(out + r * ldo + c, o);
    }
  }
}

// d2 == 1: statistics and apply in one kernel (one warp per row; the second
// pass re-reads the row, mostly from L2).  Measured against the split kernels
// (profiles/r01_ln_fused.md): forward 119 -> 87 us per step (x leaves HBM
// once), backward even (its two passes touch 3x more bytes per row than L2 can
// hold across the resident warps).  Holding the row in registers instead was
// slower (one 8-warp CTA per SM at 220 registers).
__global__ void ln_fwd_fused_kernel(const __nv_bfloat16* __restrict__ x, int64_t ldx, int64_t rows, int64_t cols,
                                    const __nv_bfloat16* __restrict__ gamma, const __nv_bfloat16* __restrict__ beta,
                                    __nv_bfloat16* __restrict__ y, int64_t ldy, float* __restrict__ saved) {
  const int lane = threadIdx.x % 32;
  for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32; r < rows;
       r += (static_cast<int64_t>(gridDim.x) * blockDim.x) / 32) {
    // shifted one-pass moments: sums of (x - K) with K = the row's first
    // element, so var = E[(x-K)^2] - E[x-K]^2 does not cancel when |mean| >> std
    const float K = __bfloat162float(x[r * ldx]);
    float s = 0.f, q = 0.f;
#pragma unroll 4
    for (int64_t c = 8 * lane; c < cols; c += 256) {
      const F8 v = ld8(x + r * ldx + c);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float t = v.v[i] - K;
        s += t;
        q += t * t;
      }
    }
    s = warp_sum(s);
    q = warp_sum(q);
    const float ms = s / static_cast<float>(cols);
    const float mean = K + ms;
    const float var = fmaxf(q / static_cast<float>(cols) - ms * ms, 0.f);
    const float rstd = rsqrtf(var + kLnEps);
#pragma unroll 4
    for (int64_t c = 8 * lane; c < cols; c += 256) {
      const F8 v = ld8(x + r * ldx + c), g = ld8(gamma + c), b = ld8(beta + c);
      F8 o;
#pragma unroll
      for (int i = 0; i < 8; ++i) o.v[i] = (v.v[i] - mean) * rstd * g.v[i] + b.v[i];
      st8(y + r * ldy + c, o);
    }
    if (lane == 0) {
      saved[2 * r] = mean;
      saved[2 * r + 1] = rstd;
    }
  }
}

__global__ void ln_bwd_fused_kernel(const __nv_bfloat16* __restrict__ dy, int64_t lddy, const __nv_bfloat16* __restrict__ x,
                                    int64_t ldx, int64_t rows, int64_t cols, const __nv_bfloat16* __restrict__ gamma,
                                    const float* __restrict__ saved, const __nv_bfloat16* res, int64_t ldres,
                                    __nv_bfloat16* out, int64_t ldo) {
  const int lane = threadIdx.x % 32;
  for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32; r < rows;
       r += (static_cast<int64_t>(gridDim.x) * blockDim.x) / 32) {
    const float mean = saved[2 * r], rstd = saved[2 * r + 1];
    float s = 0.f, q = 0.f;
#pragma unroll 4
    for (int64_t c = 8 * lane; c < cols; c += 256) {
      const F8 d = ld8(dy + r * lddy + c), v = ld8(x + r * ldx + c), g = ld8(gamma + c);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float gg = d.v[i] * g.v[i];
        s += gg;
        q += gg * (v.v[i] - mean) * rstd;
      }
    }
    const float m1 = warp_sum(s) / static_cast<float>(cols), m2 = warp_sum(q) / static_cast<float>(cols);
#pragma unroll 4
    for (int64_t c = 8 * lane; c < cols; c += 256) {
      const F8 d = ld8(dy + r * lddy + c), v = ld8(x + r * ldx + c), g = ld8(gamma + c);
      const F8 rr = ld8(res + r * ldres + c);
      F8 o;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float xh = (v.v[i] - mean) * rstd;
        o.v[i] = rr.v[i] + rstd * (d.v[i] * g.v[i] - m1 - xh * m2);
      }
      st8(out + r * ldo + c, o);
    }
  }
}

// d2 == 1, register-resident variant: one CTA of cols/16 threads per row
// (grid-stride over rows), each thread holding 16 contiguous-in-chunks
// columns of every operand, so each operand leaves HBM exactly once; the two
// row sums go through a shared-memory table (double-buffered by row parity:
// one __syncthreads per row) and every thread adds the warp partials in the
// same order (deterministic).  Needs cols % 512 == 0 and cols <= 16384.
constexpr int kRowV = 2;  // 8-column vectors per thread
__device__ __forceinline__ void block_sum2(float& s, float& q, float (*red)[2][32], int par) {
  const int lane = threadIdx.x % 32, w = threadIdx.x / 32, nw = blockDim.x / 32;
  s = warp_sum(s);
  q = warp_sum(q);
  if (lane == 0) {
    red[par][0][w] = s;
    red[par][1][w] = q;
  }
  __syncthreads();
  s = 0.f;
  q = 0.f;
  for (int i = 0; i < nw; ++i) {
    s += red[par][0][i];
    q += red[par][1][i];
  }
}

__global__ void __launch_bounds__(1024) ln_fwd_row_kernel(const __nv_bfloat16* __restrict__ x, int64_t ldx,
                                                          int64_t rows, int64_t cols,
                                                          const __nv_bfloat16* __restrict__ gamma,
                                                          const __nv_bfloat16* __restrict__ beta,
                                                          __nv_bfloat16* __restrict__ y, int64_t ldy,
                                                          float* __restrict__ saved) {
  __shared__ float red[2][2][32];
  const int64_t stride = 8 * static_cast<int64_t>(blockDim.x);
  const int64_t c0 = 8 * static_cast<int64_t>(threadIdx.x);
  F8 g[kRowV], b[kRowV];
#pragma unroll
  for (int v = 0; v < kRowV; ++v) {
    g[v] = ld8(gamma + c0 + v * stride);
    b[v] = ld8(beta + c0 + v * stride);
  }
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    // two-pass moments from the register-resident row (no extra HBM traffic):
    // mean first, then sum (x - mean)^2 -- no cancellation when |mean| >> std.
    // The two reductions use the two halves of `red`, so a row's first
    // reduction never overwrites values the previous row's second one reads.
    F8 xv[kRowV];
    float s = 0.f, z = 0.f;
#pragma unroll
    for (int v = 0; v < kRowV; ++v) {
      xv[v] = ld8(x + r * ldx + c0 + v * stride);
#pragma unroll
      for (int i = 0; i < 8; ++i) s += xv[v].v[i];
    }
    block_sum2(s, z, red, 0);
    const float mean = s / static_cast<float>(cols);
    float q = 0.f;
    z = 0.f;
#pragma unroll
    for (int v = 0; v < kRowV; ++v)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float t = xv[v].v[i] - mean;
        q += t * t;
      }
    block_sum2(q, z, red, 1);
    const float var = q / static_cast<float>(cols);
    const float rstd = rsqrtf(var + kLnEps);
#pragma unroll
    for (int v = 0; v < kRowV; ++v) {
      F8 o;
#pragma unroll
      for (int i = 0; i < 8; ++i) o.v[i] = (xv[v].v[i] - mean) * rstd * g[v].v[i] + b[v].v[i];
      st8(y + r * ldy + c0 + v * stride, o);
    }
    if (threadIdx.x == 0) {
      saved[2 * r] = mean;
      saved[2 * r + 1] = rstd;
    }
  }
}

__global__ void __launch_bounds__(1024) ln_bwd_row_kernel(const __nv_bfloat16* __restrict__ dy, int64_t lddy,
                                                          const __nv_bfloat16* __restrict__ x, int64_t ldx,
                                                          int64_t rows, int64_t cols,
                                                          const __nv_bfloat16* __restrict__ gamma,
                                                          const float* __restrict__ saved,
                                                          const __nv_bfloat16* res, int64_t ldres,
                                                          __nv_bfloat16* out, int64_t ldo) {
  __shared__ float red[2][2][32];
  const int64_t stride = 8 * static_cast<int64_t>(blockDim.x);
  const int64_t c0 = 8 * static_cast<int64_t>(threadIdx.x);
  F8 g[kRowV];
#pragma unroll
  for (int v = 0; v < kRowV; ++v) g[v] = ld8(gamma + c0 + v * stride);
  int par = 0;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x, par ^= 1) {
    const float mean = saved[2 * r], rstd = saved[2 * r + 1];
    F8 dg[kRowV], xh[kRowV];
    float s = 0.f, q = 0.f;
#pragma unroll
    for (int v = 0; v < kRowV; ++v) {
      const F8 d = ld8(dy + r * lddy + c0 + v * stride), xv = ld8(x + r * ldx + c0 + v * stride);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        dg[v].v[i] = d.v[i] * g[v].v[i];
        xh[v].v[i] = (xv.v[i] - mean) * rstd;
        s += dg[v].v[i];
        q += dg[v].v[i] * xh[v].v[i];
      }
    }
    block_sum2(s, q, red, par);
    const float m1 = s / static_cast<float>(cols), m2 = q / static_cast<float>(cols);
#pragma unroll
    for (int v = 0; v < kRowV; ++v) {
      const F8 rr = ld8(res + r * ldres + c0 + v * stride);
      F8 o;
#pragma unroll
      for (int i = 0; i < 8; ++i) o.v[i] = rr.v[i] + rstd * (dg[v].v[i] - m1 - xh[v].v[i] * m2);
      st8(out + r * ldo + c0 + v * stride, o);
    }
  }
}

bool ln_row_ok(int64_t cols) {
  static const bool on = [] {  // ATP_LN_ROW=0 keeps the warp-per-row kernels (A/B)
    const char* e = getenv("ATP_LN_ROW");
    return !(e && e[0] == '0');
  }();
  return on && cols % 512 == 0 && cols <= 16384;
}
unsigned ln_row_grid(int64_t rows, int64_t cols) {
  const int64_t per_sm = 2048 / (cols / 16);  // resident CTAs per SM by threads
  const int64_t cap = static_cast<int64_t>(num_sms()) * (per_sm > 0 ? per_sm : 1);
  return static_cast<unsigned>(rows < cap ? (rows > 0 ? rows : 1) : cap);
}

// Partial column sums over row segment blockIdx.y: part[0][seg][c] = sum dy*xhat,
// part[1][seg][c] = sum dy.  Eight columns per thread (16-byte loads, eight
// independent accumulators); rows in order, so the sums are deterministic.
__global__ void ln_param_part_kernel(const __nv_bfloat16* __restrict__ dy, int64_t lddy,
                                     const __nv_bfloat16* __restrict__ x, int64_t ldx, int64_t rows, int64_t cols,
                                     const float* __restrict__ saved, float* __restrict__ part) {
  const int64_t c = 8 * (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x);
  if (c >= cols) return;
  const int64_t per = (rows + kSegs - 1) / kSegs;
  const int64_t r0 = blockIdx.y * per, r1 = r0 + per < rows ? r0 + per : rows;
  float sg[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, sb[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 2
  for (int64_t r = r0; r < r1; ++r) {
    const F8 d = ld8(dy + r * lddy + c), v = ld8(x + r * ldx + c);
    const float mean = saved[2 * r], rstd = saved[2 * r + 1];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      sg[i] += d.v[i] * ((v.v[i] - mean) * rstd);
      sb[i] += d.v[i];
    }
  }
  float* pg = part + static_cast<int64_t>(blockIdx.y) * cols + c;
  float* pb = part + (kSegs + static_cast<int64_t>(blockIdx.y)) * cols + c;
  reinterpret_cast<float4*>(pg)[0] = make_float4(sg[0], sg[1], sg[2], sg[3]);
  reinterpret_cast<float4*>(pg)[1] = make_float4(sg[4], sg[5], sg[6], sg[7]);
  reinterpret_cast<float4*>(pb)[0] = make_float4(sb[0], sb[1], sb[2], sb[3]);
  reinterpret_cast<float4*>(pb)[1] = make_float4(sb[4], sb[5], sb[6], sb[7]);
}

// Sum the kSegs partials per column: 32 columns x 8 segment groups per CTA
// (coalesced 128-byte rows, 16 independent loads in flight per thread), then
// the 8 group sums in a fixed order, so the result stays deterministic.
constexpr int kFinCols = 32, kFinGroups = 8;
__global__ void __launch_bounds__(kFinCols* kFinGroups) ln_param_final_kernel(const float* __restrict__ part,
                                                                              int64_t cols, float* __restrict__ dgamma,
                                                                              float* __restrict__ dbeta) {
  __shared__ float red[2][kFinGroups][kFinCols];
  const int lx = threadIdx.x % kFinCols, g = threadIdx.x / kFinCols;
  const int64_t c = blockIdx.x * static_cast<int64_t>(kFinCols) + lx;
  float sg = 0.f, sb = 0.f;
  if (c < cols) {
#pragma unroll 16
    for (int s = g; s < kSegs; s += kFinGroups) {
      sg += part[s * cols + c];
      sb += part[(kSegs + s) * cols + c];
    }
  }
  red[0][g][lx] = sg;
  red[1][g][lx] = sb;
  __syncthreads();
  if (g == 0 && c < cols) {
    float tg = 0.f, tb = 0.f;
#pragma unroll
    for (int i = 0; i < kFinGroups; ++i) {
      tg += red[0][i][lx];
      tb += red[1][i][lx];
    }
    dgamma[c] = tg;
    dbeta[c] = tb;
  }
}

// [rows, p*w] (pitch ld) -> [p][rows][w]   (pack = 1), or back (pack = 0).
__global__ void block_pack_kernel(const __nv_bfloat16* __restrict__ in, __nv_bfloat16* __restrict__ out, int64_t rows,
                                  int64_t w, int p, int64_t ld, int pack) {
  const int64_t w8 = w / 8, n = rows * p * w8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c8 = i % w8, t = i / w8;
    const int64_t r = t % rows, j = t / rows;
    const int64_t blk = (j * rows + r) * w + 8 * c8, flat = r * ld + j * w + 8 * c8;
    if (pack)
      *reinterpret_cast<uint4*>(out + blk) = *reinterpret_cast<const uint4*>(in + flat);
    else
      *reinterpret_cast<uint4*>(out + flat) = *reinterpret_cast<const uint4*>(in + blk);
  }
}

}  // namespace

size_t ln_param_workspace_bytes(int64_t cols) { return static_cast<size_t>(2 * kSegs) * cols * sizeof(float); }

cudaError_t gpt_ew_launch(const EwDesc& e, cudaStream_t st) {
  using bf = __nv_bfloat16;
  const int64_t lda = e.lda > 0 ? e.lda : e.cols;
  const int64_t ldo = e.ldo > 0 ? e.ldo : e.cols;
  switch (e.kind) {
    case EW_LN_STATS:
      ln_stats_kernel<<<grid_for(e.rows), 256, 0, st>>>(static_cast<const bf*>(e.a), lda, e.rows, e.cols,
                                                        static_cast<float*>(e.out2));
      break;
    case EW_LN_APPLY:
      ln_apply_kernel<<<grid_for(e.rows), 256, 0, st>>>(
          static_cast<const bf*>(e.a), lda, e.rows, e.cols, static_cast<const float*>(e.out2),
          static_cast<float>(e.n_total), static_cast<const bf*>(e.b), static_cast<const bf*>(e.c),
          static_cast<bf*>(e.out), ldo, static_cast<float*>(e.ws));
      break;
    case EW_LN_BWD_STATS:
      ln_bwd_stats_kernel<<<grid_for(e.rows), 256, 0, st>>>(
          static_cast<const bf*>(e.a), lda, static_cast<const bf*>(e.b), e.ldb > 0 ? e.ldb : e.cols, e.rows, e.cols,
          static_cast<const bf*>(e.c), static_cast<const float*>(e.ws), static_cast<float*>(e.out2));
      break;
    case EW_LN_BWD_APPLY:
      ln_bwd_apply_kernel<<<grid_for(e.rows), 256, 0, st>>>(
          static_cast<const bf*>(e.a), lda, static_cast<const bf*>(e.b), e.ldb > 0 ? e.ldb : e.cols, e.rows, e.cols,
          static_cast<const bf*>(e.c), static_cast<const float*>(e.ws), static_cast<const float*>(e.out2),
          static_cast<float>(e.n_total), static_cast<const bf*>(e.res), e.ldres > 0 ? e.ldres : e.cols,
          static_cast<bf*>(e.out), ldo);
      break;
    case EW_LN_FWD:
      if (ln_row_ok(e.cols)) {
        ln_fwd_row_kernel<<<ln_row_grid(e.rows, e.cols), static_cast<unsigned>(e.cols / 16), 0, st>>>(
            static_cast<const bf*>(e.a), lda, e.rows, e.cols, static_cast<const bf*>(e.b), static_cast<const bf*>(e.c),
            static_cast<bf*>(e.out), ldo, static_cast<float*>(e.ws));
        break;
      }
      ln_fwd_fused_kernel<<<grid_for(e.rows), 256, 0, st>>>(
          static_cast<const bf*>(e.a), lda, e.rows, e.cols, static_cast<const bf*>(e.b), static_cast<const bf*>(e.c),
          static_cast<bf*>(e.out), ldo, static_cast<float*>(e.ws));
      break;
    case EW_LN_BWD:
      if (ln_row_ok(e.cols)) {
        ln_bwd_row_kernel<<<ln_row_grid(e.rows, e.cols), static_cast<unsigned>(e.cols / 16), 0, st>>>(
            static_cast<const bf*>(e.a), lda, static_cast<const bf*>(e.b), e.ldb > 0 ? e.ldb : e.cols, e.rows, e.cols,
            static_cast<const bf*>(e.c), static_cast<const float*>(e.ws), static_cast<const bf*>(e.res),
            e.ldres > 0 ? e.ldres : e.cols, static_cast<bf*>(e.out), ldo);
        break;
      }
      ln_bwd_fused_kernel<<<grid_for(e.rows), 256, 0, st>>>(
          static_cast<const bf*>(e.a), lda, static_cast<const bf*>(e.b), e.ldb > 0 ? e.ldb : e.cols, e.rows, e.cols,
          static_cast<const bf*>(e.c), static_cast<const float*>(e.ws), static_cast<const bf*>(e.res),
          e.ldres > 0 ? e.ldres : e.cols, static_cast<bf*>(e.out), ldo);
      break;
    case EW_LN_PARAM_GRAD: {
      float* part = static_cast<float*>(e.out2);  // workspace: ln_param_workspace_bytes(cols)
      dim3 grid(static_cast<unsigned>((e.cols / 8 + 255) / 256), kSegs);  // 8 columns per thread (cols % 8 == 0)
      ln_param_part_kernel<<<grid, 256, 0, st>>>(static_cast<const bf*>(e.a), lda, static_cast<const bf*>(e.b),
                                                 e.ldb > 0 ? e.ldb : e.cols, e.rows, e.cols,
                                                 static_cast<const float*>(e.ws), part);
      ln_param_final_kernel<<<static_cast<unsigned>((e.cols + kFinCols - 1) / kFinCols), kFinCols * kFinGroups, 0, st>>>(
          part, e.cols, static_cast<float*>(e.out), static_cast<float*>(e.res_out));
      break;
    }
    case EW_PACK:
    case EW_UNPACK: {
      const int64_t n = e.rows * e.cols / 8;  // cols = p * w
      const int64_t blocks = (n + 255) / 256, cap = static_cast<int64_t>(num_sms()) * 8;
      block_pack_kernel<<<static_cast<int>(blocks < cap ? blocks : cap), 256, 0, st>>>(
          static_cast<const bf*>(e.a), static_cast<bf*>(e.out), e.rows, e.cols / e.p, e.p,
          e.kind == EW_PACK ? lda : ldo, e.kind == EW_PACK ? 1 : 0);
      break;
    }
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace atp
