// Fused grouped all-reduce over peer memory (opt-in "fused" stages), the
// collective half of a fused GEMM -> all-reduce -> elementwise stage.
//
// PAPER.md §4.1 contrasts ATP's chunking with fusing the GEMM and its
// all-reduce; on NVSwitch both compose: the stage's GEMM (gemm_sm100.cu,
// PushArgs) already performs the reduce-scatter's data movement — each
// 128-row output tile is TMA-stored straight into the receive slot of the
// member that owns the tile's row slice and counted on that member's chunk
// counter (release, system scope).  Then, per chunk k, ONE kernel per member j
// on the communication stream (two launches: phase A, then B + C):
//
//   A. reduce: waits for chunk k's tiles from all p senders, streams its
//      slice of the p partials (and the elementwise step's side input) through
//      a shared-memory ring filled by 1-D bulk copies, sums them in member
//      order (bf16x2 adds, rounded per add like a ring's hops; for two
//      members exactly the once-rounded sum), writes the sum back in place (its own
//      slot) for the peers to pull, applies the stage's elementwise step
//      (GeLU / dGeLU / residual / stand-in core) and writes its slice of the
//      outputs; publishes `ready`;
//   B. all-gather by pull: for every other member, once it is ready, streams
//      that member's reduced slice through the same ring (bulk copies over
//      NVLink: kFusedStages x kFusedStageBytes in flight per CTA, so the pull
//      is bandwidth- not latency-bound) and applies the elementwise step on
//      the way into the local outputs;
//   C. tells every member it is done reading; CTA 0 retires only when every
//      member is done with this member's slice.
//
// NVLink bytes per member and chunk: (p-1)/p of the chunk pushed by the GEMM
// + (p-1)/p pulled = the ring all-reduce's 2(p-1)/p, with no NCCL call, no
// local partial-sum round trip through HBM for the pushed tiles, and no
// separate elementwise pass.  Peers are other GPUs' buffers mapped with CUDA
// IPC (distributed mesh) or other virtual ranks' buffers on the same GPU
// (virtual mesh).  Counters use cumulative targets computed on the host, so
// they are never reset.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "atp_internal.h"
#include "elementwise.h"
#include "fused_ar.h"
#include "gelu.cuh"
#include "sm100_ptx.cuh"

namespace atp {

namespace {

using bf = __nv_bfloat16;

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
__device__ __forceinline__ void red_release_sys(uint32_t* p) {
  asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}

// Vectors of 8 bf16 as uint4 (four bf16x2 words).  The sums and the residual
// stay packed (HADD2.BF16: the correctly rounded sum, i.e. for two bf16
// operands exactly the fp32 sum rounded once — what the unfused path stores);
// only GeLU / GeLU' go through fp32.  Unpacking every element to fp32 and back
// made these kernels ALU-bound (~190 instructions per 8-element vector).
__device__ __forceinline__ uint4 lds16(uint32_t addr) {
  uint4 u;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w) : "r"(addr));
  return u;
}
__device__ __forceinline__ uint32_t hadd2(uint32_t a, uint32_t b) {
  __nv_bfloat162 r = __hadd2(*reinterpret_cast<const __nv_bfloat162*>(&a), *reinterpret_cast<const __nv_bfloat162*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}
__device__ __forceinline__ uint4 add8(uint4 a, uint4 b) {
  return make_uint4(hadd2(a.x, b.x), hadd2(a.y, b.y), hadd2(a.z, b.z), hadd2(a.w, b.w));
}
__device__ __forceinline__ void st16(bf* p, uint4 v) { *reinterpret_cast<uint4*>(p) = v; }
__device__ __forceinline__ void unpack8(const uint4 u, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return u;
}

// The stage's elementwise step on 8 all-reduced values v at element `pos` of
// a slice whose first row is g0 (the stage output and GeLU's H are [T, W]
// with pitch W, so the element sits at g0 * W + pos); x = the step's side
// input at the same position (residual / saved U), staged in shared memory
// with v.  Writes the stage output (`out`) and the step's own output.
__device__ __forceinline__ void finish8(const FusedArArgs& a, int64_t g0, uint32_t pos, uint4 v, uint4 x) {
  const int64_t o = g0 * a.ld + pos;
  switch (a.ew_kind) {
    case EW_GELU: {  // out = U (all-reduced), ew_out = H = GeLU(U)
      float f[8];
      unpack8(v, f);
#pragma unroll
      for (int e = 0; e < 8; ++e) f[e] = gelu::gelu(f[e]);
      st16(static_cast<bf*>(a.ew_out) + o, pack8(f));
      break;
    }
    case EW_DGELU: {  // out = dU = dH * GeLU'(U)
      float f[8], u[8];
      unpack8(v, f);
      unpack8(x, u);
#pragma unroll
      for (int e = 0; e < 8; ++e) f[e] *= gelu::gelu_grad(u[e]);
      v = pack8(f);
      break;
    }
    case EW_ADD:  // out = residual + all-reduced
      v = add8(x, v);
      break;
    case EW_CORE_BWD: {  // dQ = dK = dV = dctx of the head; dQKV is [T, 3W]
      const uint32_t W = static_cast<uint32_t>(a.width), dd = static_cast<uint32_t>(a.head_dim);
      const uint32_t row = pos / W, col = pos - row * W, hd = col / dd, jj = col - hd * dd;
      bf* dst = static_cast<bf*>(a.ew_out) + (g0 + row) * a.ew_ld + hd * 3 * dd + jj;
      st16(dst, v);
      st16(dst + dd, v);
      st16(dst + 2 * dd, v);
      break;
    }
    default:
      break;
  }
  st16(static_cast<bf*>(a.out) + o, v);
}

// Stand-in core forward (ctx = Q + K + V per head): the q vector at element
// `pos` of the slice (k at +d, v at +2d), jj = its column inside the head.
// The QKV output is [T, W]; ctx is [T, W/3] and the head triple (3d columns)
// maps to d columns, so ctx's element is (pos - jj) / 3 + jj of the slice.
__device__ __forceinline__ void finish_core(const FusedArArgs& a, int64_t g0, uint32_t pos, uint32_t jj, uint4 q,
                                            uint4 k, uint4 v) {
  const int64_t d = a.head_dim;
  bf* oq = static_cast<bf*>(a.out) + g0 * a.ld + pos;
  st16(oq, q);
  st16(oq + d, k);
  st16(oq + 2 * d, v);
  st16(static_cast<bf*>(a.ew_out) + g0 * a.ew_ld + (pos - jj) / 3u + jj, add8(add8(q, k), v));
}

// One pass over the byte range [b_lo, b_hi) of `nbuf` equally laid-out
// sources, piece by piece through the shared-memory ring: thread 0 keeps
// kFusedStages pieces in flight (one bulk copy per source and piece; `full`
// mbarrier per stage with the transaction bytes); every warp runs
// process(stage, off, nbytes) on each landed piece and then arrives on the
// stage's `empty` mbarrier, so a warp moves on to the next landed piece
// without waiting for the other warps; thread 0 refills a stage once all
// warps have left it.  `consumed` counts pieces over all calls of the kernel
// (stage = count % kFusedStages, parity = (count / kFusedStages) & 1).
template <class F>
__device__ __forceinline__ void stream_pieces(uint32_t sbase, uint32_t full0, uint32_t empty0, uint32_t& consumed,
                                              int nbuf, const char* const* src, int64_t piece, int64_t b_lo,
                                              int64_t b_hi, F&& process) {
  const int np = b_hi > b_lo ? static_cast<int>((b_hi - b_lo + piece - 1) / piece) : 0;
  const uint32_t base_count = consumed;
  auto issue = [&](int q) {
    const uint32_t gq = base_count + q, st = gq % kFusedStages;
    if (gq >= kFusedStages) ptx::mbar_wait(empty0 + 8u * st, ((gq / kFusedStages) - 1) & 1u);  // previous use left
    const int64_t off = b_lo + static_cast<int64_t>(q) * piece;
    const uint32_t bytes = static_cast<uint32_t>(min(piece, b_hi - off));
    ptx::mbar_arrive_expect_tx(full0 + 8u * st, bytes * static_cast<uint32_t>(nbuf));
    for (int b = 0; b < nbuf; ++b)
      ptx::bulk_load_1d(sbase + st * kFusedStageBytes + static_cast<uint32_t>(b * piece), src[b] + off, bytes,
                        full0 + 8u * st);
  };
  if (threadIdx.x == 0)
    for (int q = 0; q < np && q < kFusedStages; ++q) issue(q);
  for (int q = 0; q < np; ++q) {
    const uint32_t st = consumed % kFusedStages;
    ptx::mbar_wait(full0 + 8u * st, (consumed / kFusedStages) & 1u);
    const int64_t off = b_lo + static_cast<int64_t>(q) * piece;
    process(sbase + st * kFusedStageBytes, off, min(piece, b_hi - off));
    __syncwarp();
    if ((threadIdx.x & 31) == 0) ptx::mbar_arrive(empty0 + 8u * st);
    if (threadIdx.x == 0 && q + kFusedStages < np) issue(q + kFusedStages);
    ++consumed;
  }
}

// PHASE 0 = A (needs only the GEMMs' tiles), PHASE 1 = B + C (needs the
// peers' phase A).  Two launches per chunk: a CTA that spins on a peer never
// holds an SM that a phase-A CTA of its own rank needs, so partially resident
// grids on different ranks cannot wait on each other in a cycle.
template <int PHASE>
__global__ void __launch_bounds__(kFusedThreads, 2) fused_ar_kernel(FusedArArgs a) {
  extern __shared__ uint8_t smem_raw[];
  const int tid = threadIdx.x, nt = blockDim.x;
  const bool core = a.ew_kind == EW_CORE_FWD;
  const bool side = a.ew_kind == EW_ADD || a.ew_kind == EW_DGELU;  // side input staged with the values
  const int64_t S = a.rows / a.p, d = a.head_dim;
  const int64_t row_bytes = a.ld * 2;
  const uint32_t sbase = (ptx::smem_u32(smem_raw) + 127u) & ~127u;
  const uint32_t full0 = sbase + kFusedStages * kFusedStageBytes, empty0 = full0 + 8u * kFusedStages;
  uint32_t* my_flags = reinterpret_cast<uint32_t*>(a.peer_base[a.me] + a.flag_off);
  const char* mine = a.peer_base[a.me] + a.part_off;
  const int64_t r0 = a.chunk * S, g0 = a.row0 + static_cast<int64_t>(a.me) * S;
  // this CTA's byte range of a slice (S rows): whole units (core: whole (q, k, v) head triples)
  const int64_t unit = core ? 3 * d * 2 : 16;
  const int64_t n_units = S * a.width * 2 / unit;
  const int64_t b_lo = n_units * blockIdx.x / gridDim.x * unit;
  const int64_t b_hi = n_units * (blockIdx.x + 1) / gridDim.x * unit;
  const int nbuf_a = a.p + (side ? 1 : 0);
  const int64_t piece = (kFusedStageBytes / nbuf_a / unit) * unit;
  const char* ewa = static_cast<const char*>(a.ew_a);
  uint32_t consumed = 0;
  // per-thread item strides in elements: generic items are 8-element vectors
  // (stride nt * 8); core items advance by nt / per whole (q, k, v) triples
  const uint32_t per = core ? static_cast<uint32_t>(d / 8) : 1u;  // ctx vectors per head triple
  const uint32_t dstep = core ? (static_cast<uint32_t>(nt) / per) * static_cast<uint32_t>(3 * d)
                              : static_cast<uint32_t>(nt) * 8u;
  if (tid == 0) {
    for (int s = 0; s < kFusedStages; ++s) {
      ptx::mbar_init(full0 + 8u * s, 1);
      ptx::mbar_init(empty0 + 8u * s, kFusedThreads / 32);
    }
    ptx::fence_barrier_init();
    if (PHASE == 0) {
      spin_geq(my_flags + a.sig_slot, a.sig_target);  // every sender's tiles of my slice have landed
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
  }
  __syncthreads();

  // ---- A. reduce my slice: the p partial slots (+ side input) staged together
  if (PHASE == 0) {
    const char* src[kMaxPush + 1];
    for (int m = 0; m < a.p; ++m) src[m] = mine + (static_cast<int64_t>(m) * a.slot_rows + r0) * row_bytes;
    if (side) src[a.p] = ewa + g0 * row_bytes;
    bf* dst = reinterpret_cast<bf*>(const_cast<char*>(src[a.me]));  // the sum goes back in place (my slot)
    stream_pieces(sbase, full0, empty0, consumed, nbuf_a, src, piece, b_lo, b_hi,
                  [&](uint32_t stg, int64_t off, int64_t nb) {
      if (core) {
        const uint32_t items = static_cast<uint32_t>(nb / unit) * per;
        const uint32_t tt0 = static_cast<uint32_t>(tid) / per, jj = (static_cast<uint32_t>(tid) - tt0 * per) * 8u;
        uint32_t e = tt0 * 3u * static_cast<uint32_t>(d) + jj;  // element in the piece
        for (uint32_t it = tid; it < items; it += nt, e += dstep) {
          const uint32_t sa = stg + 2u * e;
          uint4 q = lds16(sa), k = lds16(sa + 2 * d), v = lds16(sa + 4 * d);
          for (int m = 1; m < a.p; ++m) {  // member order: ((p0 + p1) + p2) ..., rounded per add
            const uint32_t sm = sa + static_cast<uint32_t>(m * piece);
            q = add8(q, lds16(sm));
            k = add8(k, lds16(sm + 2 * d));
            v = add8(v, lds16(sm + 4 * d));
          }
          const uint32_t pos = static_cast<uint32_t>(off / 2) + e;  // element of the slice
          bf* dq = dst + pos;  // the sum back in place, for the peers
          st16(dq, q);
          st16(dq + d, k);
          st16(dq + 2 * d, v);
          finish_core(a, g0, pos, jj, q, k, v);
        }
      } else {
        const uint32_t items = static_cast<uint32_t>(nb / 16), p0 = static_cast<uint32_t>(off / 2);
        for (uint32_t it = tid; it < items; it += nt) {
          const uint32_t sa = stg + it * 16u;
          uint4 acc = lds16(sa);
          for (int m = 1; m < a.p; ++m) acc = add8(acc, lds16(sa + static_cast<uint32_t>(m * piece)));
          st16(dst + p0 + it * 8u, acc);
          const uint4 x = side ? lds16(sa + static_cast<uint32_t>(a.p * piece)) : make_uint4(0, 0, 0, 0);
          finish8(a, g0, p0 + it * 8u, acc, x);
        }
      }
    });
  }
  if (PHASE == 0) {
    __syncthreads();
    if (tid == 0) red_release_sys(my_flags + kSigSlots + a.sig_slot);  // ready (release, cumulative via the barrier)
    return;
  }

  // ---- B. all-gather by pull: every other member's reduced slice (+ side input)
  const int nbuf_b = side ? 2 : 1;
  for (int t = 1; t < a.p; ++t) {
    const int j = (a.me + t) % a.p;
    const int64_t gj = a.row0 + static_cast<int64_t>(j) * S;
    const char* src[2] = {a.peer_base[j] + a.part_off + (static_cast<int64_t>(j) * a.slot_rows + r0) * row_bytes,
                          side ? ewa + gj * row_bytes : nullptr};
    if (tid == 0 && b_hi > b_lo) {
      spin_geq(reinterpret_cast<const uint32_t*>(a.peer_base[j] + a.flag_off) + kSigSlots + a.sig_slot,
               a.ready_target);
      asm volatile("fence.proxy.async.global;" ::: "memory");  // generic-proxy writes -> bulk-copy reads
    }
    stream_pieces(sbase, full0, empty0, consumed, nbuf_b, src, piece, b_lo, b_hi,
                  [&](uint32_t stg, int64_t off, int64_t nb) {
      if (core) {
        const uint32_t items = static_cast<uint32_t>(nb / unit) * per;
        const uint32_t tt0 = static_cast<uint32_t>(tid) / per, jj = (static_cast<uint32_t>(tid) - tt0 * per) * 8u;
        uint32_t e = tt0 * 3u * static_cast<uint32_t>(d) + jj;
        for (uint32_t it = tid; it < items; it += nt, e += dstep) {
          const uint32_t sa = stg + 2u * e;
          finish_core(a, gj, static_cast<uint32_t>(off / 2) + e, jj, lds16(sa), lds16(sa + 2 * d), lds16(sa + 4 * d));
        }
      } else {
        const uint32_t items = static_cast<uint32_t>(nb / 16), p0 = static_cast<uint32_t>(off / 2);
        for (uint32_t it = tid; it < items; it += nt) {
          const uint32_t sa = stg + it * 16u;
          const uint4 x = side ? lds16(sa + static_cast<uint32_t>(piece)) : make_uint4(0, 0, 0, 0);
          finish8(a, gj, p0 + it * 8u, lds16(sa), x);
        }
      }
    });
  }

  // ---- C. nobody reads my slice once every member's CTAs are done
  __syncthreads();
  if (tid == 0) {
    for (int m = 0; m < a.p; ++m)
      red_release_sys(reinterpret_cast<uint32_t*>(a.peer_base[m] + a.flag_off) + 2 * kSigSlots + a.sig_slot);
    if (blockIdx.x == 0) spin_geq(my_flags + 2 * kSigSlots + a.sig_slot, a.done_target);
  }
}

}  // namespace

cudaError_t fused_ar_launch(const FusedArArgs& a, cudaStream_t st) {
  constexpr int smem = kFusedStages * kFusedStageBytes + 2 * kFusedStages * 8 + 128;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(fused_ar_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(fused_ar_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  // Launched as 2-CTA clusters: the CTA-pair GEMMs need both SMs of a pair
  // free, and fused CTAs scattered one per SM pair could leave no pair for the
  // GEMM clusters whose tiles those very CTAs wait for (with every rank of a
  // virtual mesh on one GPU this deadlocked: DESIGN.md §10).  As clusters the
  // fused CTAs take whole pairs.  The kernel uses no cluster feature.
  cudaLaunchConfig_t cfg = {};
  if (a.n_ctas % 2) return cudaErrorInvalidValue;  // the ready / done targets count n_ctas CTAs
  cfg.gridDim = dim3(a.n_ctas);
  cfg.blockDim = dim3(kFusedThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute cl[1];
  cl[0].id = cudaLaunchAttributeClusterDimension;
  cl[0].val.clusterDim.x = 2;
  cl[0].val.clusterDim.y = 1;
  cl[0].val.clusterDim.z = 1;
  cfg.attrs = cl;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, fused_ar_kernel<0>, a);
  if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, fused_ar_kernel<1>, a);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace atp
