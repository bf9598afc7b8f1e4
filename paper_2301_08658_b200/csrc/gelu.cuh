// Exact-erf GeLU and its derivative for the bf16 path (reading G15, PAPER.md
// GeLU(x) = x * Phi(x)), shared by the GEMM epilogues, the post-all-reduce
// elementwise kernels and the fused all-reduce.  erf via Abramowitz & Stegun
// 7.1.26 (|error| <= 1.5e-7, fp32 level; outputs are rounded to bf16, 2^-9):
//   erf(z) = 1 - t(a1 + t(a2 + t(a3 + t(a4 + t a5)))) e^{-z^2},  t = 1/(1 + p z), z >= 0,
// with MUFU reciprocal and exp2 (one instruction each, ~1 ulp).  With
// z = |x|/sqrt 2, e^{-z^2} = e^{-x^2/2} is also phi(x) sqrt(2 pi), so
// GeLU'(x) = Phi(x) + x phi(x) reuses it.  The fp32 check mode keeps erff.
#pragma once
#include <cuda_runtime.h>

namespace atp {
namespace gelu {

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
struct ErfExp {
  float erf_abs;  // erf(|x|/sqrt 2)
  float e;        // exp(-x^2/2)
};
__device__ __forceinline__ ErfExp erf_as(float x) {
  const float z = fabsf(x) * 0.70710678118654752f;
  const float t = rcp_approx(fmaf(0.3275911f, z, 1.0f));
  const float poly =
      t * fmaf(t, fmaf(t, fmaf(t, fmaf(t, 1.061405429f, -1.453152027f), 1.421413741f), -0.284496736f), 0.254829592f);
  const float e = ex2_approx(-0.72134752044448170f * x * x);  // exp(-x^2/2) = 2^(-x^2 / (2 ln 2))
  return {1.0f - poly * e, e};
}
__device__ __forceinline__ float gelu(float x) {
  const ErfExp r = erf_as(x);
  return 0.5f * x * (1.0f + copysignf(r.erf_abs, x));
}
__device__ __forceinline__ float gelu_grad(float x) {
  const ErfExp r = erf_as(x);
  return fmaf(0.5f, 1.0f + copysignf(r.erf_abs, x), x * 0.39894228040143268f * r.e);
}

}  // namespace gelu
}  // namespace atp
