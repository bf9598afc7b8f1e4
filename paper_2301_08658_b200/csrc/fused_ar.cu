// Fused grouped all-reduce over peer memory (opt-in "fused" stages).
//
// One kernel per chunk k of a communicating stage, on the communication
// stream, replaces ncclAllReduce(chunk k) + the post-all-reduce elementwise
// step.  Every member of the mesh-dimension group has written its partial
// sums of the stage into its peer-visible ("symmetric") buffer with the
// signalled GEMM, which counts finished tiles per chunk.  With p members and
// the chunk's rows cut into p row slices (slice j owned by member j):
//
//   1. wait until every member's tile counter for chunk k is complete;
//   2. reduce-scatter: member j sums slice j of all p partial buffers (fixed
//      member order, fp32) and writes the bf16 sum in place into slice j of
//      its own buffer, then bumps its `ready` counter;
//   3. all-gather by pull: every member copies each slice j from member j's
//      buffer into its own output rows and applies the stage's elementwise
//      step (GeLU / dGeLU / residual / attention stand-in core) on the way;
//   4. every CTA bumps every member's `done` counter; CTA 0 waits for all
//      members' CTAs, so when the kernel retires nobody reads this member's
//      buffer any more and the next GEMM may overwrite it.
//
// Bytes moved over NVLink per member: 2(p-1)/p of the chunk (ring-optimal),
// with the elementwise pass fused into the gather.  Peers are other GPUs'
// buffers mapped with CUDA IPC (distributed mesh) or other virtual ranks'
// buffers on the same GPU (virtual mesh).  Counters use cumulative targets
// computed on the host, so they are never reset.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "atp_internal.h"
#include "elementwise.h"
#include "fused_ar.h"
#include "gelu.cuh"

namespace atp {

namespace {

__device__ __forceinline__ float gelu_f(float x) { return gelu::gelu(x); }  // bf16 path (gelu.cuh)
__device__ __forceinline__ float gelu_grad_f(float x) { return gelu::gelu_grad(x); }

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// cyclic >= (targets wrap at 2^32)
__device__ __forceinline__ void spin_geq(const uint32_t* p, uint32_t target) {
  while (static_cast<int32_t>(ld_acquire_sys(p) - target) < 0) {
  }
}

__device__ __forceinline__ void load8(const __nv_bfloat16* p, float (&f)[8]) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ void store8(__nv_bfloat16* p, const float (&f)[8]) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}

__global__ void __launch_bounds__(512) fused_ar_kernel(FusedArArgs a) {
  using bf = __nv_bfloat16;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t w8 = a.width / 8;
  auto part = [&](int m, int64_t row) {  // member m's partial row (global row index)
    return reinterpret_cast<bf*>(a.peer_base[m] + a.part_off) + row * a.ld;
  };
  auto slice_begin = [&](int j) { return a.row0 + (a.rows * j) / a.p; };

  // ---- 1. every member's GEMM has finished chunk k
  if (tid == 0)
    for (int m = 0; m < a.p; ++m) spin_geq(reinterpret_cast<const uint32_t*>(a.peer_base[m] + a.flag_off) + a.sig_slot, a.sig_target);
  __syncthreads();

  // ---- 2. reduce-scatter: my slice, summed over members in member order, in place
  {
    const int64_t r0 = slice_begin(a.me), r1 = slice_begin(a.me + 1);
    const int64_t n = (r1 - r0) * w8;
    for (int64_t i = blockIdx.x * (int64_t)nt + tid; i < n; i += (int64_t)gridDim.x * nt) {
      const int64_t row = r0 + i / w8, c8 = (i % w8) * 8;
      float acc[8], v[8];
      load8(part(0, row) + c8, acc);
      for (int m = 1; m < a.p; ++m) {
        load8(part(m, row) + c8, v);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += v[e];
      }
      store8(part(a.me, row) + c8, acc);
    }
  }
  __syncthreads();
  uint32_t* my_flags = reinterpret_cast<uint32_t*>(a.peer_base[a.me] + a.flag_off);
  if (tid == 0) {
    __threadfence_system();
    atomicAdd(my_flags + kSigSlots + a.sig_slot, 1u);  // ready
  }

  // ---- 3. all-gather by pull + the stage's elementwise step: a flat
  // grid-stride loop over (row, 8-column vector) pairs of each slice.  For the
  // stand-in core the loop runs over ctx vectors and pulls the q, k, v vectors
  // of the head (each is written exactly once), so no intra-row sync is needed.
  const bool core_fwd = a.ew_kind == EW_CORE_FWD;
  const int64_t vec_per_row = core_fwd ? a.ew_width / 8 : w8;
  for (int j = 0; j < a.p; ++j) {
    if (tid == 0)
      spin_geq(reinterpret_cast<const uint32_t*>(a.peer_base[j] + a.flag_off) + kSigSlots + a.sig_slot, a.ready_target);
    __syncthreads();
    const int64_t r0 = slice_begin(j), r1 = slice_begin(j + 1);
    const int64_t n = (r1 - r0) * vec_per_row;
    for (int64_t i = blockIdx.x * (int64_t)nt + tid; i < n; i += (int64_t)gridDim.x * nt) {
      const int64_t row = r0 + i / vec_per_row, c8 = (i % vec_per_row) * 8;
      bf* orow = static_cast<bf*>(a.out) + row * a.ld;
      const bf* src = part(j, row);
      if (core_fwd) {
        const int64_t hd = c8 / a.head_dim, jj = c8 % a.head_dim;
        const int64_t q = hd * 3 * a.head_dim + jj;
        float x[8], k[8], v[8];
        load8(src + q, x);
        load8(src + q + a.head_dim, k);
        load8(src + q + 2 * a.head_dim, v);
        store8(orow + q, x);
        store8(orow + q + a.head_dim, k);
        store8(orow + q + 2 * a.head_dim, v);
#pragma unroll
        for (int e = 0; e < 8; ++e) x[e] = (x[e] + k[e]) + v[e];
        store8(static_cast<bf*>(a.ew_out) + row * a.ew_ld + c8, x);
        continue;
      }
      float v[8];
      load8(src + c8, v);  // the all-reduced (bf16) values
      if (a.ew_kind == EW_GELU) {
        float h[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) h[e] = gelu_f(v[e]);
        store8(static_cast<bf*>(a.ew_out) + row * a.ew_ld + c8, h);
      } else if (a.ew_kind == EW_DGELU) {
        float u[8];
        load8(static_cast<const bf*>(a.ew_a) + row * a.ew_lda + c8, u);
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] *= gelu_grad_f(u[e]);
      } else if (a.ew_kind == EW_ADD) {
        float x[8];
        load8(static_cast<const bf*>(a.ew_a) + row * a.ew_lda + c8, x);
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = x[e] + v[e];
      } else if (a.ew_kind == EW_CORE_BWD) {
        // dQ = dK = dV = dctx of the head (row-local)
        const int64_t hd = c8 / a.head_dim, jj = c8 % a.head_dim;
        bf* dst = static_cast<bf*>(a.ew_out) + row * a.ew_ld + hd * 3 * a.head_dim + jj;
        store8(dst, v);
        store8(dst + a.head_dim, v);
        store8(dst + 2 * a.head_dim, v);
      }
      store8(orow + c8, v);
    }
  }

  // ---- 4. nobody reads my buffer once every member's CTAs are done
  __syncthreads();
  if (tid == 0) {
    __threadfence_system();
    for (int m = 0; m < a.p; ++m)
      atomicAdd(reinterpret_cast<uint32_t*>(a.peer_base[m] + a.flag_off) + 2 * kSigSlots + a.sig_slot, 1u);
    if (blockIdx.x == 0) spin_geq(my_flags + 2 * kSigSlots + a.sig_slot, a.done_target);
  }
}

}  // namespace

cudaError_t fused_ar_launch(const FusedArArgs& a, cudaStream_t st) {
  fused_ar_kernel<<<a.n_ctas, 512, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace atp
