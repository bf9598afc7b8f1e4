// HBM-bound elementwise steps of the ATP block that cannot live in a GEMM
// epilogue because an all-reduce sits between the GEMM and them (the GEMM
// output is a Partial(SUM); GeLU and the residual are applied to the SUM):
//   gelu_rows     H = GeLU(U)                      F10 (exact erf)
//   dgelu_rows    dU = dH * GeLU'(U)   (in place)  B2
//   add_rows      out = a + out        (in place)  residuals F7/F12/B3/B6
//   core_fwd      ctx = Q + K + V per head         F5 (stand-in core, G20)
//   core_bwd      dQ = dK = dV = dctx              B5
//   colsum        db[n] = sum_t dY[t, n]  (fp32, deterministic, no workspace)
//   group_sum     virtual-mesh all-reduce: sum of p member buffers, in
//                 ascending coordinate order, written back to every member
// All kernels move 16 B per thread per access (8 bf16) and use grid-stride
// loops with a grid sized to a multiple of the SM count.
#include <cuda_bf16.h>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "atp_internal.h"
#include "attention.h"
#include "elementwise.h"
#include "gelu.cuh"

namespace atp {

namespace {

// bf16 path: the MUFU-based exact-erf form (gelu.cuh; erff made these kernels
// ALU-bound at ~2.4 TB/s); fp32 check mode: erff / expf.
template <class T>
__device__ __forceinline__ float gelu_f(float x) {
  if constexpr (sizeof(T) == 2) return gelu::gelu(x);
  return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f));
}
template <class T>
__device__ __forceinline__ float gelu_grad_f(float x) {
  if constexpr (sizeof(T) == 2) return gelu::gelu_grad(x);
  return 0.5f * (1.0f + erff(x * 0.70710678118654752f)) + x * 0.39894228040143268f * expf(-0.5f * x * x);
}

struct V8 {
  float f[8];
};
__device__ __forceinline__ V8 ld8(const float* p) {
  const float4 a = reinterpret_cast<const float4*>(p)[0];
  const float4 b = reinterpret_cast<const float4*>(p)[1];
  V8 r;
  r.f[0] = a.x; r.f[1] = a.y; r.f[2] = a.z; r.f[3] = a.w;
  r.f[4] = b.x; r.f[5] = b.y; r.f[6] = b.z; r.f[7] = b.w;
  return r;
}
__device__ __forceinline__ void st8(float* p, const V8& v) {
  reinterpret_cast<float4*>(p)[0] = make_float4(v.f[0], v.f[1], v.f[2], v.f[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(v.f[4], v.f[5], v.f[6], v.f[7]);
}
__device__ __forceinline__ V8 ld8(const __nv_bfloat16* p) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
  V8 r;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    r.f[2 * i] = f.x;
    r.f[2 * i + 1] = f.y;
  }
  return r;
}
__device__ __forceinline__ void st8(__nv_bfloat16* p, const V8& v) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v.f[2 * i], v.f[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}

// Elementwise over a dense [rows, cols] matrix (cols % 8 == 0), n8 = rows*cols/8.
template <class T>
__global__ void gelu_kernel(const T* __restrict__ u, T* __restrict__ h, int64_t n8) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    V8 v = ld8(u + 8 * i);
#pragma unroll
    for (int j = 0; j < 8; ++j) v.f[j] = gelu_f<T>(v.f[j]);
    st8(h + 8 * i, v);
  }
}

template <class T>
__global__ void dgelu_kernel(T* __restrict__ dh, const T* __restrict__ u, int64_t n8) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    V8 g = ld8(dh + 8 * i);
    V8 x = ld8(u + 8 * i);
#pragma unroll
    for (int j = 0; j < 8; ++j) g.f[j] *= gelu_grad_f<T>(x.f[j]);
    st8(dh + 8 * i, g);
  }
}

template <class T>
__global__ void add_kernel(const T* __restrict__ a, T* __restrict__ out, int64_t n8) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    V8 x = ld8(a + 8 * i);
    V8 y = ld8(out + 8 * i);
#pragma unroll
    for (int j = 0; j < 8; ++j) y.f[j] += x.f[j];
    st8(out + 8 * i, y);
  }
}

// ctx[t, hd*d + j] = qkv[t, hd*3d + j] + qkv[t, hd*3d + d + j] + qkv[t, hd*3d + 2d + j]
// One thread per 8 ctx columns; d % 8 == 0.
template <class T>
__global__ void core_fwd_kernel(const T* __restrict__ qkv, T* __restrict__ ctx, int64_t rows, int heads, int d) {
  const int w8 = heads * d / 8;
  const int64_t n = rows * w8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / w8;
    const int c8 = static_cast<int>(i % w8) * 8;
    const int hd = c8 / d, j = c8 % d;
    const T* src = qkv + t * (int64_t)(3 * heads * d) + hd * 3 * d + j;
    V8 q = ld8(src), k = ld8(src + d), v = ld8(src + 2 * d);
#pragma unroll
    for (int e = 0; e < 8; ++e) q.f[e] = (q.f[e] + k.f[e]) + v.f[e];
    st8(ctx + t * (int64_t)(heads * d) + c8, q);
  }
}

template <class T>
__global__ void core_bwd_kernel(const T* __restrict__ dctx, T* __restrict__ dqkv, int64_t rows, int heads, int d) {
  const int w8 = heads * d / 8;
  const int64_t n = rows * w8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / w8;
    const int c8 = static_cast<int>(i % w8) * 8;
    const int hd = c8 / d, j = c8 % d;
    const V8 v = ld8(dctx + t * (int64_t)(heads * d) + c8);
    T* dst = dqkv + t * (int64_t)(3 * heads * d) + hd * 3 * d + j;
    st8(dst, v);
    st8(dst + d, v);
    st8(dst + 2 * d, v);
  }
}

// db[c] = sum_t x[t, c], deterministic and workspace-free.  A cluster of
// kColsumSplit CTAs shares one 128-column strip: CTA s sums its contiguous
// row range (8 warps, 4 columns per lane, rows in order per warp, warps added
// in order), then CTA 0 adds the kColsumSplit partials in rank order through
// distributed shared memory.
constexpr int kColsumSplit = 8;
constexpr int kColsumWarps = 8;
__device__ __forceinline__ float4 ld4f(const __nv_bfloat16* p) {
  const uint2 v = *reinterpret_cast<const uint2*>(p);
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.y));
  return make_float4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ float4 ld4f(const float* p) { return *reinterpret_cast<const float4*>(p); }

template <class T>
__global__ void __launch_bounds__(kColsumWarps * 32) colsum_kernel(const T* __restrict__ x, float* __restrict__ out,
                                                                  int64_t rows, int cols) {
  namespace cg = cooperative_groups;
  __shared__ float4 part[kColsumWarps][32];
  __shared__ float4 total[32];
  cg::cluster_group cluster = cg::this_cluster();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int s = static_cast<int>(cluster.block_rank());
  const int c4 = blockIdx.x * 128 + 4 * lane;
  const int64_t per = (rows + kColsumSplit - 1) / kColsumSplit;
  const int64_t r0 = s * per, r1 = min(rows, r0 + per);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (c4 < cols) {
    int64_t r = r0 + warp;
    for (; r + 3 * kColsumWarps < r1; r += 4 * kColsumWarps) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = ld4f(x + (r + u * kColsumWarps) * cols + c4);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc.x += v[u].x;
        acc.y += v[u].y;
        acc.z += v[u].z;
        acc.w += v[u].w;
      }
    }
    for (; r < r1; r += kColsumWarps) {
      const float4 v = ld4f(x + r * cols + c4);
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
  }
  part[warp][lane] = acc;
  __syncthreads();
  if (warp == 0) {
    float4 t = part[0][lane];
    for (int w = 1; w < kColsumWarps; ++w) {
      t.x += part[w][lane].x;
      t.y += part[w][lane].y;
      t.z += part[w][lane].z;
      t.w += part[w][lane].w;
    }
    total[lane] = t;
  }
  cluster.sync();
  if (s == 0 && warp == 0 && c4 < cols) {
    float4 t = total[lane];
    for (int r = 1; r < kColsumSplit; ++r) {
      const float4* remote = cluster.map_shared_rank(total, r);
      const float4 u = remote[lane];
      t.x += u.x;
      t.y += u.y;
      t.z += u.z;
      t.w += u.w;
    }
    *reinterpret_cast<float4*>(out + c4) = t;
  }
  cluster.sync();  // keep every CTA's shared memory alive until rank 0 has read it
}

template <class T>
__global__ void group_sum_kernel(GroupSumArgs g, int64_t n8) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    V8 acc = ld8(static_cast<const T*>(g.buf[0]) + 8 * i);
    for (int r = 1; r < g.p; ++r) {
      V8 v = ld8(static_cast<const T*>(g.buf[r]) + 8 * i);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc.f[j] += v.f[j];
    }
    for (int r = 0; r < g.p; ++r) st8(static_cast<T*>(g.buf[r]) + 8 * i, acc);
  }
}

int ew_grid(int64_t n) {
  const int64_t per = 256;
  int64_t blocks = (n + per - 1) / per;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  return blocks < 1 ? 1 : static_cast<int>(blocks);
}

}  // namespace

template <class T>
cudaError_t ew_launch_t(const EwDesc& e, cudaStream_t st) {
  const int64_t n = e.rows * e.cols;
  switch (e.kind) {
    case EW_GELU:
      gelu_kernel<T><<<ew_grid(n / 8), 256, 0, st>>>((const T*)e.a, (T*)e.out, n / 8);
      break;
    case EW_DGELU:
      dgelu_kernel<T><<<ew_grid(n / 8), 256, 0, st>>>((T*)e.out, (const T*)e.a, n / 8);
      break;
    case EW_ADD:
      add_kernel<T><<<ew_grid(n / 8), 256, 0, st>>>((const T*)e.a, (T*)e.out, n / 8);
      break;
    case EW_CORE_FWD:
      core_fwd_kernel<T><<<ew_grid(n / 8), 256, 0, st>>>((const T*)e.a, (T*)e.out, e.rows, e.heads,
                                                         static_cast<int>(e.cols / e.heads));
      break;
    case EW_CORE_BWD:
      core_bwd_kernel<T><<<ew_grid(n / 8), 256, 0, st>>>((const T*)e.a, (T*)e.out, e.rows, e.heads,
                                                         static_cast<int>(e.cols / e.heads));
      break;
    case EW_COLSUM: {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(static_cast<unsigned>((e.cols + 127) / 128), kColsumSplit);
      cfg.blockDim = dim3(kColsumWarps * 32);
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 1;
      attr[0].val.clusterDim.y = kColsumSplit;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      return cudaLaunchKernelEx(&cfg, colsum_kernel<T>, (const T*)e.a, (float*)e.out, e.rows, static_cast<int>(e.cols));
    }
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t ew_launch(const EwDesc& e, cudaStream_t st) {
  if (e.kind == EW_ATTN_FWD)
    return attn_fwd_launch(e.a, e.lda, static_cast<int>(e.rows), e.seq, e.heads, e.causal, e.out, e.ldo,
                           static_cast<float*>(e.out2), st, e.ws, static_cast<size_t>(e.n_total));
  if (e.kind == EW_ATTN_BWD)
    return attn_bwd_launch(e.a, e.lda, e.b, e.ldb, static_cast<const float*>(e.out2), e.res, e.ldres,
                           static_cast<int>(e.rows), e.seq, e.heads, e.causal, e.out, e.ldo, e.ws, st);
  if (e.kind >= EW_LN_STATS) return gpt_ew_launch(e, st);
  return e.dtype == 1 ? ew_launch_t<float>(e, st) : ew_launch_t<__nv_bfloat16>(e, st);
}

cudaError_t group_sum_launch(const GroupSumArgs& g, int64_t n, int dtype, cudaStream_t st) {
  if (dtype == 1)
    group_sum_kernel<float><<<ew_grid(n / 8), 256, 0, st>>>(g, n / 8);
  else
    group_sum_kernel<__nv_bfloat16><<<ew_grid(n / 8), 256, 0, st>>>(g, n / 8);
  return cudaGetLastError();
}

}  // namespace atp
