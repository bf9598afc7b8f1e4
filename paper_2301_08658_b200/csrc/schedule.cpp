// Schedule builders: the per-rank op lists of the ATP linears and blocks.
//
// Chunk pipeline (§4.1 Fig. 7; reading G14): the rows of
// every activation are cut into `c` chunks; each linear ("stage") is emitted
// breadth-first over the chunks — GEMM(k), all-reduce(k) — on two streams, and
// chunk k of stage s+1 waits only for the all-reduce of chunk k of stage s.
// Host enqueue order is the op order below, i.e. each all-reduce is submitted
// before the GEMM it should overlap (the reason for the paper's
// CUDA_DEVICE_MAX_CONNECTIONS=1).
//
// Backward (§4.2): per linear, the dX GEMMs are chunked and each
// chunk's all-reduce overlaps the next chunk; the dW GEMM runs once over all
// T rows right after that linear's dX chunks, overlapping their all-reduces
// (dW feeds no collective, so chunking it would only add fp32 read-modify-write
// traffic).
//
// Bias placement (reading G16): a bias is added exactly once per reduction
// group — fused into the GEMM epilogue of the coordinate-0 rank before the
// all-reduce, or unconditionally when the reducing dimension has size 1.
// Elementwise steps that follow an all-reduce (GeLU, dGeLU, residual, core)
// are separate HBM-bound kernels; when the reducing dimension has size 1 they
// are fused into the GEMM epilogue instead (EPI_RESID / EPI_BIAS_GELU /
// EPI_DGELU).
#include <string>
#include <vector>

#include "runtime.h"
#include "schedule.h"

namespace atp {

namespace {

using bf16 = __nv_bfloat16;

inline const char* cptr(const void* p, int64_t off_elems) {
  return static_cast<const char*>(p) + off_elems * 2;
}
inline char* mptr(void* p, int64_t off_elems) { return static_cast<char*>(p) + off_elems * 2; }

struct Builder {
  Sched s;
  RankView rv;
  std::string err;
  int chunks = 1;
  int64_t T = 0, Mc = 0;
  std::vector<int> pend;                // per chunk: event the next stage's chunk must wait on
  std::vector<std::vector<EwDesc>> def;  // per chunk: deferred prologue ops

  Builder(const RankView& v, int64_t rows, int c) : rv(v), chunks(c), T(rows), Mc(rows / c) {
    pend.assign(c, -1);
    def.assign(c, {});
  }
  int ev() { return s.n_events++; }

  Op& push(OpKind k, int stream) {
    s.ops.emplace_back();
    Op& o = s.ops.back();
    o.kind = k;
    o.stream = stream;
    return o;
  }
  static void add_wait(Op& o, int e) {
    if (e >= 0) o.waits[o.n_waits++] = e;
  }
  // Emit chunk k's pending wait + deferred prologue ops on the compute stream.
  // Returns the wait that is still unconsumed (if no prologue op carried it).
  int prologue(int k) {
    int w = pend[k];
    pend[k] = -1;
    for (const EwDesc& e : def[k]) {
      Op& o = push(OP_EW, 0);
      o.e = e;
      add_wait(o, w);
      w = -1;
    }
    def[k].clear();
    return w;
  }
  bool gemm(const void* A, int64_t lda, bool a_mn, const void* B, int64_t ldb, bool b_mn, int64_t M, int64_t N,
            int64_t K, int epi, const EpiParams& ep, int wait, int record, int bn = 0) {
    Op& o = push(OP_GEMM, 0);
    o.g.bn = bn;
    o.g.max_ctas = rv.gemm_ctas;
    o.g.epi = epi;
    o.g.ep = ep;
    const char* m = gemm_prepare(o.g, A, lda, a_mn, B, ldb, b_mn, static_cast<int>(M), static_cast<int>(N),
                                 static_cast<int>(K));
    if (m) {
      err = m;
      return false;
    }
    add_wait(o, wait);
    o.record = record;
    return true;
  }
  void allreduce(int dim, void* ptr, int64_t count, int wait, int record) {
    Op& o = push(OP_AR, 1);
    o.ar_dim = dim;
    o.ar_ptr = ptr;
    o.ar_count = count;
    add_wait(o, wait);
    o.record = record;
  }
  void ew_now(const EwDesc& e, int wait = -1) {
    Op& o = push(OP_EW, 0);
    o.e = e;
    add_wait(o, wait);
  }
  int dim_size(int dim) const { return dim == 1 ? rv.d1 : rv.d2; }
  bool coord0(int dim) const { return (dim == 1 ? rv.i1 : rv.i2) == 0; }

  // One forward linear stage over all chunks: out_k = in_k W (+bias), then the
  // grouped all-reduce over `dim` (skipped when that dimension has size 1).
  // `fused` = epilogue to use when no all-reduce follows.  `after_ar(k)` =
  // deferred elementwise ops of chunk k once the sum is available.
  template <class AfterAR, class FusedEp>
  bool fwd_stage(int dim, const void* in, int64_t in_w, const void* w, int64_t out_w, const void* bias, void* out,
                 int fused_epi, FusedEp fused_ep, AfterAR after_ar) {
    const bool comm = dim_size(dim) > 1;
    for (int k = 0; k < chunks; ++k) {
      const int wait = prologue(k);
      EpiParams ep;
      int epi = EPI_BF16;
      ep.C = mptr(out, k * Mc * out_w);
      ep.ldc = out_w;
      if (comm) {
        ep.bias = coord0(dim) ? static_cast<const bf16*>(bias) : nullptr;
      } else {
        ep.bias = static_cast<const bf16*>(bias);
        epi = fused_epi;
        fused_ep(k, ep);
      }
      const int e = comm ? ev() : -1;
      if (!gemm(cptr(in, k * Mc * in_w), in_w, false, w, out_w, true, Mc, out_w, in_w, epi, ep, wait, e))
        return false;
      if (comm) {
        const int r = ev();
        allreduce(dim, ep.C, Mc * out_w, e, r);
        pend[k] = r;
        after_ar(k);
      }
    }
    return true;
  }

  // One backward linear stage: dx_k = dy_k W^T then all-reduce over `dim`
  // (the conjugate dimension); dW = X^T dY over all T rows afterwards.
  template <class AfterAR, class FusedEp>
  bool bwd_stage(int dim, const void* dy, int64_t dy_w, const void* w, int64_t x_w, void* dx, int fused_epi,
                 FusedEp fused_ep, AfterAR after_ar) {
    const bool comm = dim_size(dim) > 1;
    for (int k = 0; k < chunks; ++k) {
      const int wait = prologue(k);
      EpiParams ep;
      int epi = EPI_BF16;
      ep.C = mptr(dx, k * Mc * x_w);
      ep.ldc = x_w;
      if (!comm) {
        epi = fused_epi;
        fused_ep(k, ep);
      }
      const int e = comm ? ev() : -1;
      // dx_k [Mc, x_w] = dy_k [Mc, dy_w] * W[x_w, dy_w]^T: A K-major, B = W stored [x_w, dy_w] K-major
      if (!gemm(cptr(dy, k * Mc * dy_w), dy_w, false, w, dy_w, false, Mc, x_w, dy_w, epi, ep, wait, e))
        return false;
      if (comm) {
        const int r = ev();
        allreduce(dim, ep.C, Mc * x_w, e, r);
        pend[k] = r;
        after_ar(k);
      }
    }
    return true;
  }
  // dW[x_w, dy_w] (fp32) = X[T, x_w]^T dY[T, dy_w]  (both MN-major), + dbias = colsum(dY)
  bool dw(const void* x, int64_t x_w, const void* dy, int64_t dy_w, float* dwp, float* dbias) {
    EpiParams ep;
    ep.C = dwp;
    ep.ldc = dy_w;
    if (dwp != nullptr && !gemm(x, x_w, true, dy, dy_w, true, x_w, dy_w, T, EPI_F32, ep, -1, -1)) return false;
    if (dbias != nullptr) {
      EwDesc e;
      e.kind = EW_COLSUM;
      e.out = dbias;
      e.a = dy;
      e.rows = T;
      e.cols = dy_w;
      ew_now(e);
    }
    return true;
  }
  void flush() {
    for (int k = 0; k < chunks; ++k) {
      int w = prologue(k);
      (void)w;  // a trailing all-reduce with no consumer is joined by the executor
    }
  }
  static EwDesc ew(int kind, void* out, const void* a, int64_t rows, int64_t cols, int heads = 1) {
    EwDesc e;
    e.kind = kind;
    e.out = out;
    e.a = a;
    e.rows = rows;
    e.cols = cols;
    e.heads = heads;
    return e;
  }
};

auto no_fuse = [](int, EpiParams&) {};
auto no_after = [](int) {};

}  // namespace

// ---------------------------------------------------------------- linears
int build_linear_fwd(const RankView& rv, bool colfirst, const LinearFwd& a, int64_t M, int64_t K, int64_t N,
                     int chunks, Sched& out) {
  Builder b(rv, M, chunks);
  const int dim = colfirst ? 2 : 1;
  const int64_t in_w = colfirst ? K / rv.d2 : K / rv.d1;
  const int64_t out_w = colfirst ? N / rv.d1 : N / rv.d2;
  if (!b.fwd_stage(dim, a.x, in_w, a.w, out_w, a.bias, a.y, EPI_BF16, no_fuse, no_after)) {
    set_error(b.err);
    return 2;
  }
  b.flush();
  out = std::move(b.s);
  return 0;
}

int build_linear_bwd(const RankView& rv, bool colfirst, const LinearBwd& a, int64_t M, int64_t K, int64_t N,
                     int chunks, Sched& out) {
  Builder b(rv, M, chunks);
  const int dim = colfirst ? 1 : 2;  // conjugate dimension ("f3 ... on the second dimension in backward")
  const int64_t x_w = colfirst ? K / rv.d2 : K / rv.d1;
  const int64_t dy_w = colfirst ? N / rv.d1 : N / rv.d2;
  if (!b.bwd_stage(dim, a.dy, dy_w, a.w, x_w, a.dx, EPI_BF16, no_fuse, no_after) ||
      !b.dw(a.x, x_w, a.dy, dy_w, a.dw, a.dbias)) {
    set_error(b.err);
    return 2;
  }
  b.flush();
  out = std::move(b.s);
  return 0;
}

// ---------------------------------------------------------------- layer blocks
int build_layer(const RankView& rv, const LayerParts& p, int64_t T, int64_t h, int64_t F, int64_t heads,
                int chunks, Sched& out) {
  Builder b(rv, T, chunks);
  const int64_t Mc = T / chunks;
  const int64_t hc = h / rv.d2;       // activation column block
  const int64_t h1 = h / rv.d1;       // ctx width / Out input
  const int64_t q1 = 3 * h / rv.d1;   // local QKV width
  const int64_t F1 = F / rv.d1;       // local FFN width
  const int64_t hl = heads / rv.d1;   // local heads
  const int d1 = rv.d1, d2 = rv.d2;
  auto rowsof = [&](const void* base, int k, int64_t w) { return cptr(base, k * Mc * w); };
  auto mrowsof = [&](void* base, int k, int64_t w) { return mptr(base, k * Mc * w); };
  auto fail = [&]() {
    set_error(b.err);
    return 2;
  };

  if (p.attn_fwd) {
    const atp_attn_fwd_args& a = *p.attn_fwd;
    // F3/F4: QKV column-first, all-reduce on dim 2 (f1); F5 core deferred
    if (!b.fwd_stage(2, a.x, hc, a.wqkv, q1, a.bqkv, a.qkv, EPI_BF16, no_fuse, no_after)) return fail();
    for (int k = 0; k < chunks; ++k)
      b.def[k].push_back(Builder::ew(EW_CORE_FWD, mrowsof(a.ctx, k, h1), rowsof(a.qkv, k, q1), Mc, h1, (int)hl));
    // F6/F7: Out row-first, all-reduce on dim 1 (f2), residual Y1 = X + .
    if (!b.fwd_stage(
            1, a.ctx, h1, a.wo, hc, a.bo, a.y, EPI_RESID,
            [&](int k, EpiParams& ep) {
              ep.aux = static_cast<const bf16*>(static_cast<const void*>(rowsof(a.x, k, hc)));
              ep.ldaux = hc;
            },
            [&](int k) { b.def[k].push_back(Builder::ew(EW_ADD, mrowsof(a.y, k, hc), rowsof(a.x, k, hc), Mc, hc)); }))
      return fail();
  }
  if (p.mlp_fwd) {
    const atp_mlp_fwd_args& a = *p.mlp_fwd;
    // F8/F9/F10: FC1 column-first, all-reduce on dim 2 (f3), U saved, H = GeLU(U)
    if (!b.fwd_stage(
            2, a.x, hc, a.w1, F1, a.b1, a.u, EPI_BIAS_GELU,
            [&](int k, EpiParams& ep) {
              ep.C2 = mrowsof(a.h_act, k, F1);
              ep.ldc2 = F1;
            },
            [&](int k) {
              b.def[k].push_back(Builder::ew(EW_GELU, mrowsof(a.h_act, k, F1), rowsof(a.u, k, F1), Mc, F1));
            }))
      return fail();
    // F11/F12: FC2 row-first, all-reduce on dim 1 (f4), Z = X + .
    if (!b.fwd_stage(
            1, a.h_act, F1, a.w2, hc, a.b2, a.z, EPI_RESID,
            [&](int k, EpiParams& ep) {
              ep.aux = static_cast<const bf16*>(static_cast<const void*>(rowsof(a.x, k, hc)));
              ep.ldaux = hc;
            },
            [&](int k) { b.def[k].push_back(Builder::ew(EW_ADD, mrowsof(a.z, k, hc), rowsof(a.x, k, hc), Mc, hc)); }))
      return fail();
  }
  if (p.mlp_bwd) {
    const atp_mlp_bwd_args& a = *p.mlp_bwd;
    // B1: dH = dZ W2^T, all-reduce on dim 2 (conjugate of f4); dU = dH * GeLU'(U)
    if (!b.bwd_stage(
            2, a.dz, hc, a.w2, F1, a.ws_dh, EPI_DGELU,
            [&](int k, EpiParams& ep) {
              ep.aux = static_cast<const bf16*>(static_cast<const void*>(rowsof(a.u, k, F1)));
              ep.ldaux = F1;
            },
            [&](int k) {
              b.def[k].push_back(Builder::ew(EW_DGELU, mrowsof(a.ws_dh, k, F1), rowsof(a.u, k, F1), Mc, F1));
            }))
      return fail();
    if (!b.dw(a.h_act, F1, a.dz, hc, a.dw2, a.db2)) return fail();
    // B3: dX1 = dU W1^T, all-reduce on dim 1 (conjugate of f3); dX1 += dZ (residual)
    if (!b.bwd_stage(
            1, a.ws_dh, F1, a.w1, hc, a.dx, EPI_RESID,
            [&](int k, EpiParams& ep) {
              ep.aux = static_cast<const bf16*>(static_cast<const void*>(rowsof(a.dz, k, hc)));
              ep.ldaux = hc;
            },
            [&](int k) { b.def[k].push_back(Builder::ew(EW_ADD, mrowsof(a.dx, k, hc), rowsof(a.dz, k, hc), Mc, hc)); }))
      return fail();
    // dW1 needs every chunk's dU, which the B3 prologues completed
    if (!b.dw(a.x, hc, a.ws_dh, F1, a.dw1, a.db1)) return fail();
  }
  if (p.attn_bwd) {
    const atp_attn_bwd_args& a = *p.attn_bwd;
    // dbo / dWo need the complete dY: flush its deferred residuals first
    // (they are the prologue of B4's chunks anyway, emitted in chunk order)
    // B4: dctx = dY Wo^T, all-reduce on dim 2 (conjugate of f2); dQKV = expand(dctx)
    if (!b.bwd_stage(2, a.dy, hc, a.wo, h1, a.ws_dctx, EPI_BF16, no_fuse, no_after)) return fail();
    for (int k = 0; k < chunks; ++k)
      b.def[k].push_back(
          Builder::ew(EW_CORE_BWD, mrowsof(a.ws_dqkv, k, q1), rowsof(a.ws_dctx, k, h1), Mc, h1, (int)hl));
    if (!b.dw(a.ctx, h1, a.dy, hc, a.dwo, a.dbo)) return fail();
    // B6: dX = dQKV Wqkv^T, all-reduce on dim 1 (conjugate of f1); dX += dY (residual)
    if (!b.bwd_stage(
            1, a.ws_dqkv, q1, a.wqkv, hc, a.dx, EPI_RESID,
            [&](int k, EpiParams& ep) {
              ep.aux = static_cast<const bf16*>(static_cast<const void*>(rowsof(a.dy, k, hc)));
              ep.ldaux = hc;
            },
            [&](int k) { b.def[k].push_back(Builder::ew(EW_ADD, mrowsof(a.dx, k, hc), rowsof(a.dy, k, hc), Mc, hc)); }))
      return fail();
    if (!b.dw(a.x, hc, a.ws_dqkv, q1, a.dwqkv, a.dbqkv)) return fail();
  }
  b.flush();
  (void)d1;
  (void)d2;
  out = std::move(b.s);
  return 0;
}

}  // namespace atp
