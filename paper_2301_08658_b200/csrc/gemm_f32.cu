// fp32 check-mode GEMM (ATP_FP32): C[M,N] = A[M,K] * B[N,K]^T on the CUDA
// cores with fp32 FMA accumulation — the same operand arrangements, fused
// epilogues and chunk signalling as the tcgen05 kernel, so the whole sharded
// schedule can be checked against the fp64 oracle at <= 1e-4 (north_star).
// This is a correctness mode; the product path is the bf16 tcgen05 kernel.
//
// 128x128 output tile per 256-thread CTA, 8x8 outputs per thread, K in steps
// of 8 staged through shared memory.  Tiles are numbered chunk by chunk when
// signalling (see gemm_sm100.cu), one CTA per tile.
#include <cuda_runtime.h>

#include <cstdint>

#include "atp_internal.h"

namespace atp {

namespace {

constexpr int TB = 128;  // tile rows / cols
constexpr int TK = 8;

__device__ __forceinline__ float gelu_f(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }
__device__ __forceinline__ float gelu_grad_f(float x) {
  return 0.5f * (1.0f + erff(x * 0.70710678118654752f)) + x * 0.39894228040143268f * expf(-0.5f * x * x);
}

__global__ void __launch_bounds__(256) gemm_f32_kernel(const float* __restrict__ A, int64_t lda, int a_mn,
                                                       const float* __restrict__ B, int64_t ldb, int b_mn, int M,
                                                       int N, int K, int epi, EpiParams ep, uint32_t* sig,
                                                       int sig_rows, const uint32_t* gate, uint32_t gate_target) {
  __shared__ float As[TK][TB + 4];
  __shared__ float Bs[TK][TB + 4];
  const int num_m = (M + TB - 1) / TB, num_n = (N + TB - 1) / TB;
  const int mt_chunk = sig_rows > 0 ? sig_rows / TB : num_m;
  // chunk-major tile order (row-major inside a chunk)
  const int tile = blockIdx.x;
  const int chunk = tile / (mt_chunk * num_n);
  const int r = tile - chunk * mt_chunk * num_n;
  const int mt = chunk * mt_chunk + r / num_n, nt = r % num_n;
  const int m0 = mt * TB, n0 = nt * TB;
  const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
  if (gate != nullptr) {
    if (tid == 0) {
      uint32_t v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gate + chunk) : "memory");
      } while (static_cast<int32_t>(v - gate_target) < 0);
    }
    __syncthreads();
  }
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  for (int k0 = 0; k0 < K; k0 += TK) {
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const int e = tid + 256 * l;  // 1024 elements of each 128 x 8 slice
      const int mm = e % TB, kk = e / TB;
      const int gm = m0 + mm, gk = k0 + kk;
      float va = 0.f, vb = 0.f;
      if (gm < M && gk < K) va = a_mn ? A[static_cast<int64_t>(gk) * lda + gm] : A[static_cast<int64_t>(gm) * lda + gk];
      const int gn = n0 + mm;
      if (gn < N && gk < K) vb = b_mn ? B[static_cast<int64_t>(gk) * ldb + gn] : B[static_cast<int64_t>(gn) * ldb + gk];
      As[kk][mm] = va;
      Bs[kk][mm] = vb;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[8], b[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = As[kk][ty * 8 + i];
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = Bs[kk][tx * 8 + j];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }

  const float* bias = static_cast<const float*>(ep.bias);
  const float* aux = static_cast<const float*>(ep.aux);
  float* C = static_cast<float*>(ep.C);
  float* C2 = static_cast<float*>(ep.C2);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int row = m0 + ty * 8 + i;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int col = n0 + tx * 8 + j;
      if (col >= N) continue;
      float v = acc[i][j];
      if (bias != nullptr) v += bias[col];
      if (epi == EPI_RESID) v += aux[static_cast<int64_t>(row) * ep.ldaux + col];
      if (epi == EPI_DGELU) v *= gelu_grad_f(aux[static_cast<int64_t>(row) * ep.ldaux + col]);
      C[static_cast<int64_t>(row) * ep.ldc + col] = v;
      if (epi == EPI_BIAS_GELU) C2[static_cast<int64_t>(row) * ep.ldc2 + col] = gelu_f(v);
    }
  }
  if (sig != nullptr) {
    __syncthreads();
    if (tid == 0) {
      __threadfence_system();
      atomicAdd(sig + chunk, 1u);
    }
  }
}

}  // namespace

const char* gemm_prepare_f32(GemmDesc& d, const void* A, int64_t lda, bool a_mn, const void* B, int64_t ldb, bool b_mn,
                             int M, int N, int K) {
  if (M <= 0 || N <= 0 || K <= 0) return "gemm(fp32): M, N, K must be positive";
  d.dtype = 1;
  d.M = M;
  d.N = N;
  d.K = K;
  d.a_mn = a_mn;
  d.b_mn = b_mn;
  d.bn = TB;
  d.cg = 1;
  d.A = A;
  d.B = B;
  d.lda = lda;
  d.ldb = ldb;
  return nullptr;
}

cudaError_t gemm_launch_f32(const GemmDesc& d, cudaStream_t st) {
  const int tiles = ((d.M + TB - 1) / TB) * ((d.N + TB - 1) / TB);
  gemm_f32_kernel<<<tiles, 256, 0, st>>>(static_cast<const float*>(d.A), d.lda, d.a_mn ? 1 : 0,
                                         static_cast<const float*>(d.B), d.ldb, d.b_mn ? 1 : 0, d.M, d.N, d.K, d.epi,
                                         d.ep, d.sig, d.sig_rows, d.gate, d.gate_target);
  return cudaGetLastError();
}

}  // namespace atp
