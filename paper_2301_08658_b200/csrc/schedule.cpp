// Schedule builders: the per-rank op lists of the ATP linears and blocks.
//
// Chunk-based overlapping (§4.1 Fig. 7; reading G14): the
// token rows are cut into `c` chunks and the all-reduce of chunk k overlaps the
// computation of the later chunks.  A "stage" is one linear (GEMM + grouped
// all-reduce).  Three ways to emit a stage:
//
//  * no communication (the reducing mesh dimension has size 1): one GEMM over
//    all T rows with the following elementwise step fused into its epilogue;
//
//  * SIGNALLED (default when the chunk rows are a multiple of the tile rows):
//    ONE persistent GEMM over all T rows whose tiles run chunk by chunk; each
//    CTA-tile bumps a per-chunk counter once its output is globally visible.
//    The communication stream waits for chunk k's counter (cuStreamWaitValue32),
//    all-reduces chunk k and applies chunk k's post-all-reduce elementwise step
//    (GeLU / residual / core / dGeLU).  So chunk k's all-reduce overlaps the
//    GEMM's later chunks without cutting the GEMM into c small launches that
//    cannot fill 148 SMs; the next stage's GEMM starts once the last chunk is
//    reduced.  B200-native replacement for the paper's per-chunk kernel calls;
//
//  * PER-CHUNK fallback: c GEMM launches (breadth-first over chunks) on the
//    compute stream with event hand-off to the communication stream; chunk k
//    of stage s+1 waits only on chunk k's all-reduce of stage s.
//
// Backward (§4.2): the dX GEMM is chunked (signalled) and each
// linear's dW GEMM over all T rows is enqueued right after it, before the
// communication ops, so it runs while the dX chunks are all-reduced (dW feeds
// no collective; chunking it would only add fp32 read-modify-write traffic).
//
// Host enqueue order = op order below: every all-reduce is submitted before
// the compute that should overlap it, and every wait refers to an op submitted
// earlier, which keeps the order valid for CUDA_DEVICE_MAX_CONNECTIONS=1
// (P:345).
//
// Bias placement (reading G16): a bias is added exactly once per reduction
// group — in the GEMM epilogue of the coordinate-0 rank before the all-reduce,
// or unconditionally when the reducing dimension has size 1.
#include <cstdlib>
#include <string>
#include <vector>

#include "runtime.h"
#include "schedule.h"
#include "attention.h"

namespace atp {

namespace {

using bf16 = __nv_bfloat16;

// element size of the schedule being built (2 = bf16, 4 = fp32 check mode)
thread_local int g_esz = 2;
inline const char* cptr(const void* p, int64_t off_elems) {
  return static_cast<const char*>(p) + off_elems * g_esz;
}
inline char* mptr(void* p, int64_t off_elems) { return static_cast<char*>(p) + off_elems * g_esz; }

using EwList = std::vector<EwDesc>;

// Where the post-all-reduce elementwise step of a signalled (NCCL) stage runs:
// 1 (default) = ONE full-T launch on the compute stream once the stage's last
// chunk is all-reduced, right before the next stage's GEMM; 0 = per chunk on
// the communication stream (ATP_EW_COMPUTE=0, A/B runs).  Per chunk, the
// elementwise kernels share the SMs with the running GEMM (a persistent grid
// that leaves them few resources) and pile up behind it: measured with the
// collectives elided at cfg 4 (4,2), c = 4, the adds alone took 0.43-0.60 ms
// per step instead of 0.09-0.11 ms as full-width launches, and the compute
// stream idled 0.23-0.33 ms waiting for that backlog
// (profiles/r02_trace_42_cap*.txt).  The all-reduce of chunk k still overlaps
// the GEMM's later chunks either way.
bool ew_compute() {
  static const bool on = [] {
    const char* e = getenv("ATP_EW_COMPUTE");
    return !(e && e[0] == '0');
  }();
  return on;
}

// ATP_AUX_COLSUM=0 keeps the bias-gradient column sums on the compute stream (A/B runs).
bool aux_colsum() {
  static const bool on = [] {
    const char* e = getenv("ATP_AUX_COLSUM");
    return !(e && e[0] == '0');
  }();
  return on;
}

struct Builder {
  Sched s;
  RankView rv;
  std::string err;
  int chunks = 1;
  int64_t T = 0, Mc = 0;
  int next_slot = 0;
  std::vector<int> pend;    // per chunk: event the next compute op of that chunk must wait on
  std::vector<EwList> def;  // per chunk: deferred elementwise ops (per-chunk mode)

  int dtype = 0;  // 0 = bf16, 1 = fp32 check mode

  Builder(const RankView& v, int64_t rows, int c, int dt) : rv(v), chunks(c), T(rows), Mc(rows / c), dtype(dt) {
    pend.assign(c, -1);
    def.assign(c, {});
    g_esz = dt == 1 ? 4 : 2;
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
    if (e < 0) return;
    for (int i = 0; i < o.n_waits; ++i)
      if (o.waits[i] == e) return;
    o.waits[o.n_waits++] = e;
  }
  // Chunk k's pending wait + deferred ops on the compute stream; returns the
  // wait still unconsumed (no deferred op carried it).
  int prologue(int k) {
    int w = pend[k];
    pend[k] = -1;
    for (const EwDesc& e : def[k]) {
      Op& o = push(OP_EW, 0);
      o.e = e;
      o.e.dtype = dtype;
      add_wait(o, w);
      w = -1;
    }
    def[k].clear();
    return w;
  }
  // Every chunk's prologue; returns the distinct unconsumed waits.  An event
  // some deferred op on the compute stream already waited for is satisfied for
  // everything behind it on that stream (one signalled stage hands ALL chunks
  // the same last-all-reduce event): dropping it leaves the GEMM without a
  // stream wait, so it may use programmatic dependent launch.
  std::vector<int> prologue_all() {
    std::vector<int> w, consumed;
    for (int k = 0; k < chunks; ++k) {
      const int pk = pend[k];
      const bool had_def = !def[k].empty();
      int e = prologue(k);
      if (had_def && pk >= 0) consumed.push_back(pk);
      bool seen = false;
      for (int x : w) seen |= (x == e);
      for (int x : consumed) seen |= (x == e);
      if (e >= 0 && !seen) w.push_back(e);
    }
    return w;
  }
  Op* gemm(const void* A, int64_t lda, bool a_mn, const void* B, int64_t ldb, bool b_mn, int64_t M, int64_t N,
           int64_t K, int epi, const EpiParams& ep, const std::vector<int>& waits, int record) {
    Op& o = push(OP_GEMM, 0);
    o.g.max_ctas = rv.gemm_ctas;
    o.g.epi = epi;
    o.g.ep = ep;
    const char* m = dtype == 1 ? gemm_prepare_f32(o.g, A, lda, a_mn, B, ldb, b_mn, static_cast<int>(M),
                                                  static_cast<int>(N), static_cast<int>(K))
                               : gemm_prepare(o.g, A, lda, a_mn, B, ldb, b_mn, static_cast<int>(M),
                                              static_cast<int>(N), static_cast<int>(K));
    if (m) {
      err = m;
      return nullptr;
    }
    for (int w : waits) add_wait(o, w);
    o.record = record;
    return &o;
  }
  void allreduce(int dim, void* ptr, int64_t count, int wait, int record) {
    Op& o = push(OP_AR, 1);
    o.ar_dim = dim;
    o.ar_ptr = ptr;
    o.ar_count = count;
    o.ar_dtype = dtype;
    add_wait(o, wait);
    o.record = record;
  }
  void ew(const EwDesc& e, int stream, int wait = -1) {
    Op& o = push(OP_EW, stream);
    o.e = e;
    o.e.dtype = dtype;
    add_wait(o, wait);
  }
  int dim_size(int dim) const { return dim == 1 ? rv.d1 : rv.d2; }
  bool coord0(int dim) const { return (dim == 1 ? rv.i1 : rv.i2) == 0; }

  // One linear stage.  out[T, out_w] = in[T, in_w] * W (+bias), B given as
  // W^T-free storage (b_mn) — i.e. forward: W stored [in_w, out_w]; backward
  // dX: W stored [out_w(x_w), in_w(dy_w)] read K-major.  `after_ar(k, rows0,
  // nrows)` returns the elementwise ops that must follow the all-reduce of the
  // given row range; `fused(ep)` configures the epilogue used when no
  // all-reduce follows (epi kind `fused_epi`); `extra()` emits compute-stream
  // work (the dW GEMMs) that should overlap this stage's communication.
  // Chunk gates of the previous stage (signalled / fused stages publish one per
  // chunk after its all-reduce and elementwise step).
  int gate_slot = -1;
  int sym_region = 0;  // fused stages alternate between the two partial regions
  // The next stage reads only call inputs (the first backward stage reads dZ):
  // it waits for nothing of the previous stage (joined by the executor at the end).
  bool next_independent = false;

  // Waits for this stage's full-T GEMM: either the previous stage's chunk gates
  // (the GEMM's producer waits per chunk; no stream wait) or the usual events.
  // Returns the gate slot to use (-1 = not gated).
  int stage_entry(int64_t out_w, std::vector<int>& waits) {
    int bn = 128, cg = 1;
    if (dtype == 0) gemm_plan_tile(static_cast<int>(T), static_cast<int>(out_w), &bn, &cg);
    if (rv.gate_ok && dtype == 0 && gate_slot >= 0 && chunks > 1 && Mc % (128 * cg) == 0) {
      for (int k = 0; k < chunks; ++k) pend[k] = -1;  // the gates replace the stream waits
      const int g = gate_slot;
      gate_slot = -1;
      return g;
    }
    gate_slot = -1;
    waits = prologue_all();
    return -1;
  }
  // Pending deferred elementwise steps are not needed by an independent stage:
  // emit them on the communication stream (behind the all-reduces they
  // follow, so the compute stream does not wait for them) and drop the waits.
  void flush_to_comm() {
    for (int k = 0; k < chunks; ++k) {
      int w = pend[k];
      for (const EwDesc& e : def[k]) {
        ew(e, 1, w);
        w = -1;
      }
      def[k].clear();
      pend[k] = -1;
    }
  }
  void gate_gemm(Op* g, int gslot) {
    if (gslot < 0) return;
    g->gate_slot0 = gslot;
    g->g.sig_rows = static_cast<int>(Mc);
  }
  // After chunk k's all-reduce and elementwise step: publish gate k.
  void publish_gate(int gslot0, int k) {
    if (!rv.gate_ok) return;  // nobody waits on gates
    Op& o = push(OP_SIGNAL, 1);
    o.sig_slot = gslot0 + k;
  }

  // One linear stage.  out[T, out_w] = in[T, in_w] * W (+bias), B given as
  // W^T-free storage (b_mn) — i.e. forward: W stored [in_w, out_w]; backward
  // dX: W stored [out_w(x_w), in_w(dy_w)] read K-major.  `after_ar(k, rows0,
  // nrows)` returns the elementwise ops that must follow the all-reduce of the
  // given row range; `fused(ep)` configures the epilogue used when no
  // all-reduce follows (epi kind `fused_epi`); `extra()` emits compute-stream
  // work (the dW GEMMs) that should overlap this stage's communication.
  template <class AfterAR, class Fused, class Extra>
  bool stage(int dim, const void* in, int64_t in_w, const void* w, int64_t ldw, bool b_mn, int64_t out_w, const void* bias,
             void* out, int fused_epi, Fused fused, AfterAR after_ar, Extra extra) {
    const bool comm = dim_size(dim) > 1;
    if (next_independent) {
      // consumed by THIS stage whatever way it is emitted (the per-chunk branch
      // below never calls stage_entry): the previous stage's deferred steps go
      // to the communication stream and nothing here waits for them
      next_independent = false;
      gate_slot = -1;
      flush_to_comm();
    }
    int bn = 128, cg = 1;  // fp32 check mode: 128 x 128 tiles
    if (dtype == 0) gemm_plan_tile(static_cast<int>(T), static_cast<int>(out_w), &bn, &cg);
    if (!comm) {
      // ---- no all-reduce: one full-T GEMM, elementwise step fused into its epilogue
      std::vector<int> waits;
      const int gslot = stage_entry(out_w, waits);
      EpiParams ep;
      ep.C = out;
      ep.ldc = out_w;
      ep.bias = bias;
      fused(ep, 0, T);
      Op* g = gemm(in, in_w, false, w, ldw, b_mn, T, out_w, in_w, fused_epi, ep, waits, -1);
      if (!g) return false;
      gate_gemm(g, gslot);
      return extra();
    }
    const void* bias_here = coord0(dim) ? bias : nullptr;
    // fused GEMM -> reduce-scatter -> all-gather: each member's slice of a chunk
    // (S = Mc / p rows) must be whole 128-row CTA tiles, and every receive slot
    // row a whole number of 16-byte vectors
    const int p_grp = dim_size(dim);
    const bool fused_ok = rv.sym_base != nullptr && dtype == 0 && Mc % (128 * cg) == 0 && p_grp <= kMaxPush &&
                          (Mc / p_grp) % 128 == 0 && (out_w * 2) % 16 == 0 &&
                          static_cast<size_t>(T) * out_w * 2 <= rv.sym_part_bytes && next_slot + chunks <= kGateBase;
    const bool signalled_ok = rv.signalled && rv.sig_buf != nullptr && chunks > 1 && Mc % (128 * cg) == 0 &&
                              next_slot + chunks <= kGateBase;
    if (fused_ok || signalled_ok) {
      // ---- ONE GEMM over all T rows with per-chunk tile counters; per chunk on
      // the communication stream: the all-reduce (NCCL after a counter wait, or
      // the fused peer-memory kernel) + elementwise step, then the chunk gate.
      std::vector<int> waits;
      const int gslot_in = stage_entry(out_w, waits);
      const int64_t part_off = fused_ok ? static_cast<int64_t>(sym_region) * rv.sym_part_bytes : 0;
      if (fused_ok) sym_region ^= 1;
      EpiParams ep;
      ep.C = fused_ok ? static_cast<void*>(rv.sym_base + part_off) : out;
      ep.ldc = out_w;
      ep.bias = bias_here;
      Op* g = gemm(in, in_w, false, w, ldw, b_mn, T, out_w, in_w, EPI_BF16, ep, waits, -1);
      if (!g) return false;
      gate_gemm(g, gslot_in);
      const int slot0 = next_slot;
      const int gslot0 = kGateBase + next_slot;
      next_slot += chunks;
      g->g.sig = rv.sig_buf + slot0;
      g->g.sig_rows = static_cast<int>(Mc);
      const uint32_t per_chunk = static_cast<uint32_t>((Mc / 128) * ((out_w + g->g.bn - 1) / g->g.bn));
      if (fused_ok) {
        // the GEMM stores slice j of every chunk into member j's receive slot for
        // this rank: [T/p rows, out_w] at part_off + me * (T/p) * out_w * 2
        PushArgs& pa = g->g.push;
        const int di = dim - 1, me = rv.me_in[di];
        const int64_t slot_rows = T / p_grp;
        pa.p = p_grp;
        pa.slice_rows = static_cast<int>(Mc / p_grp);
        for (int j = 0; j < p_grp; ++j) {
          char* pb = rv.peers[di][j];
          if (pb == nullptr || !make_tmap_out(&pa.tm[j], pb + part_off + me * slot_rows * out_w * 2, 2, slot_rows,
                                              out_w, out_w, 32)) {
            err = "fused stage: receive-slot tensor map";
            return false;
          }
          pa.sig[j] = reinterpret_cast<uint32_t*>(pb + 2 * rv.sym_part_bytes) + slot0;
        }
      }
      if (!extra()) return false;
      const EwList post = fused_ok ? after_ar(0, 0, T) : EwList{};  // base pointers of the fused step
      // NCCL stage, not gated: the elementwise step runs once over all T rows
      // on the compute stream before the next stage (ew_compute()).
      const bool ew_deferred = !fused_ok && !rv.gate_ok && ew_compute();
      for (int k = 0; k < chunks; ++k) {
        if (fused_ok) {
          Op& o = push(OP_FUSED_AR, 1);
          o.ar_dim = dim;
          o.ar_count = Mc * out_w;
          o.sig_inc = per_chunk;
          FusedArArgs& f = o.far;
          f.part_off = part_off;
          f.flag_off = 2 * static_cast<int64_t>(rv.sym_part_bytes);
          f.ld = out_w;
          f.width = out_w;
          f.row0 = k * Mc;
          f.rows = Mc;
          f.chunk = k;
          f.slot_rows = T / p_grp;
          f.sig_slot = slot0 + k;
          f.out = out;
          f.n_ctas = fused_ctas();
          if (!post.empty()) {
            const EwDesc& e = post[0];
            f.ew_kind = e.kind;
            f.ew_out = e.out;
            f.ew_a = e.a;
            f.ew_ld = e.kind == EW_CORE_BWD ? 3 * e.cols : e.cols;
            f.ew_lda = e.cols;
            f.ew_width = e.cols;
            f.head_dim = e.cols / e.heads;
          }
        } else {
          Op& wsig = push(OP_WAITSIG, 1);
          wsig.sig_slot = slot0 + k;
          wsig.sig_inc = per_chunk;
          allreduce(dim, mptr(out, k * Mc * out_w), Mc * out_w, -1, -1);
          if (!ew_deferred)
            for (const EwDesc& e : after_ar(k, k * Mc, Mc)) ew(e, 1);
        }
        publish_gate(gslot0, k);
      }
      const int last = ev();
      s.ops.back().record = last;
      for (int k = 0; k < chunks; ++k) pend[k] = last;
      if (ew_deferred) def[0] = after_ar(0, 0, T);
      gate_slot = rv.gate_ok ? gslot0 : -1;
      return true;
    }
    // ---- per-chunk stage: c GEMM launches, event hand-off per chunk
    gate_slot = -1;
    for (int k = 0; k < chunks; ++k) {
      const int wait = prologue(k);
      EpiParams ep;
      ep.C = mptr(out, k * Mc * out_w);
      ep.ldc = out_w;
      ep.bias = bias_here;
      const int e = ev();
      if (!gemm(cptr(in, k * Mc * in_w), in_w, false, w, ldw, b_mn, Mc, out_w, in_w, EPI_BF16, ep, {wait}, e))
        return false;
      const int r = ev();
      allreduce(dim, ep.C, Mc * out_w, e, r);
      pend[k] = r;
      for (const EwDesc& d : after_ar(k, k * Mc, Mc)) def[k].push_back(d);
    }
    return extra();
  }

  // Event marking "everything enqueued on the compute stream so far is done"
  // (reuses the last compute op's record event); -1 if there is none.
  int mark_compute() {
    for (auto it = s.ops.rbegin(); it != s.ops.rend(); ++it) {
      if (it->stream != 0) continue;
      if (it->record < 0) it->record = ev();
      return it->record;
    }
    return -1;
  }

  // dW[x_w, dy_w] (fp32) = X[T, x_w]^T dY[T, dy_w]  (both MN-major), + dbias = colsum(dY).
  // The column sum is HBM-bound and nothing downstream needs it: it runs on the
  // auxiliary stream, gated on the compute stream having produced dY, so it
  // overlaps the compute-bound dW GEMM instead of sitting between GEMMs.
  bool dw(const void* x, int64_t x_w, const void* dy, int64_t dy_w, float* dwp, float* dbias) {
    EpiParams ep;
    ep.C = dwp;
    ep.ldc = dy_w;
    if (dbias != nullptr) {
      EwDesc e;
      e.kind = EW_COLSUM;
      e.out = dbias;
      e.a = dy;
      e.rows = T;
      e.cols = dy_w;
      ew(e, aux_colsum() ? 2 : 0, mark_compute());
    }
    if (dwp != nullptr && !gemm(x, x_w, true, dy, dy_w, true, x_w, dy_w, T, EPI_F32, ep, {}, -1)) return false;
    return true;
  }

  // Remaining deferred work; a trailing all-reduce with no consumer is joined
  // by the executor.
  void flush() { prologue_all(); }

  static EwDesc ewd(int kind, void* out, const void* a, int64_t rows, int64_t cols, int heads = 1) {
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

auto no_fuse = [](EpiParams&, int64_t, int64_t) {};
auto no_after = [](int, int64_t, int64_t) { return EwList{}; };
auto no_extra = []() { return true; };

}  // namespace

// ---------------------------------------------------------------- linears
int build_linear_fwd(const RankView& rv, bool colfirst, const LinearFwd& a, int64_t M, int64_t K, int64_t N,
                     int chunks, int dtype, Sched& out) {
  Builder b(rv, M, chunks, dtype);
  const int dim = colfirst ? 2 : 1;
  const int64_t in_w = colfirst ? K / rv.d2 : K / rv.d1;
  const int64_t out_w = colfirst ? N / rv.d1 : N / rv.d2;
  if (!b.stage(dim, a.x, in_w, a.w, out_w, true, out_w, a.bias, a.y, EPI_BF16, no_fuse, no_after, no_extra)) {
    set_error(b.err);
    return 2;
  }
  b.flush();
  out = std::move(b.s);
  return 0;
}

int build_linear_bwd(const RankView& rv, bool colfirst, const LinearBwd& a, int64_t M, int64_t K, int64_t N,
                     int chunks, int dtype, Sched& out) {
  Builder b(rv, M, chunks, dtype);
  const int dim = colfirst ? 1 : 2;  // conjugate dimension ("f3 ... on the second dimension in backward")
  const int64_t x_w = colfirst ? K / rv.d2 : K / rv.d1;
  const int64_t dy_w = colfirst ? N / rv.d1 : N / rv.d2;
  // dx [M, x_w] = dy [M, dy_w] * W[x_w, dy_w]^T: B = W stored [x_w, dy_w], K-major
  if (!b.stage(dim, a.dy, dy_w, a.w, dy_w, false, x_w, nullptr, a.dx, EPI_BF16, no_fuse, no_after,
               [&]() { return b.dw(a.x, x_w, a.dy, dy_w, a.dw, a.dbias); })) {
    set_error(b.err);
    return 2;
  }
  b.flush();
  out = std::move(b.s);
  return 0;
}

// ---------------------------------------------------------------- layer blocks
// Emit the forward (fwd) or backward (!fwd) blocks of one layer into `b`.
// `first_bwd`: this is the first backward block of the pipeline (its first
// stage reads only dZ and saved activations, so it waits for nothing of the
// forward tail).
static bool emit_layer(Builder& b, const RankView& rv, const LayerParts& p, bool fwd, bool first_bwd, int64_t T,
                       int64_t h, int64_t F, int64_t heads) {
  const int64_t hc = h / rv.d2;      // activation column block
  const int64_t h1 = h / rv.d1;      // ctx width / Out input
  const int64_t q1 = 3 * h / rv.d1;  // local QKV width
  const int64_t F1 = F / rv.d1;      // local FFN width
  const int hl = static_cast<int>(heads / rv.d1);  // local heads
  auto rows = [](const void* base, int64_t r0, int64_t w) { return cptr(base, r0 * w); };
  auto mrows = [](void* base, int64_t r0, int64_t w) { return mptr(base, r0 * w); };
  auto aux = [](const void* p) { return static_cast<const void*>(p); };
  auto fail = [&]() { return false; };
  using E = Builder;

  if (fwd && p.attn_fwd) {
    const atp_attn_fwd_args& a = *p.attn_fwd;
    // F3/F4: QKV column-first, all-reduce on dim 2 (f1); F5 core after the sum
    if (!b.stage(2, a.x, hc, a.wqkv, q1, true, q1, a.bqkv, a.qkv, EPI_BF16, no_fuse,
                 [&](int, int64_t r0, int64_t n) {
                   return EwList{E::ewd(EW_CORE_FWD, mrows(a.ctx, r0, h1), rows(a.qkv, r0, q1), n, h1, hl)};
                 },
                 [&]() {
                   if (rv.d2 == 1) b.ew(E::ewd(EW_CORE_FWD, a.ctx, a.qkv, T, h1, hl), 0);
                   return true;
                 }))
      return fail();
    // F6/F7: Out row-first, all-reduce on dim 1 (f2), residual Y1 = X + .
    if (!b.stage(1, a.ctx, h1, a.wo, hc, true, hc, a.bo, a.y, EPI_RESID,
                 [&](EpiParams& ep, int64_t, int64_t) {
                   ep.aux = aux(a.x);
                   ep.ldaux = hc;
                 },
                 [&](int, int64_t r0, int64_t n) {
                   return EwList{E::ewd(EW_ADD, mrows(a.y, r0, hc), rows(a.x, r0, hc), n, hc)};
                 },
                 no_extra))
      return fail();
  }
  if (fwd && p.mlp_fwd) {
    const atp_mlp_fwd_args& a = *p.mlp_fwd;
    // F8/F9/F10: FC1 column-first, all-reduce on dim 2 (f3), U saved, H = GeLU(U)
    if (!b.stage(2, a.x, hc, a.w1, F1, true, F1, a.b1, a.u, EPI_BIAS_GELU,
                 [&](EpiParams& ep, int64_t, int64_t) {
                   ep.C2 = a.h_act;
                   ep.ldc2 = F1;
                 },
                 [&](int, int64_t r0, int64_t n) {
                   return EwList{E::ewd(EW_GELU, mrows(a.h_act, r0, F1), rows(a.u, r0, F1), n, F1)};
                 },
                 no_extra))
      return fail();
    // F11/F12: FC2 row-first, all-reduce on dim 1 (f4), Z = X + .
    if (!b.stage(1, a.h_act, F1, a.w2, hc, true, hc, a.b2, a.z, EPI_RESID,
                 [&](EpiParams& ep, int64_t, int64_t) {
                   ep.aux = aux(a.x);
                   ep.ldaux = hc;
                 },
                 [&](int, int64_t r0, int64_t n) {
                   return EwList{E::ewd(EW_ADD, mrows(a.z, r0, hc), rows(a.x, r0, hc), n, hc)};
                 },
                 no_extra))
      return fail();
  }
  if (!fwd && p.mlp_bwd) {
    const atp_mlp_bwd_args& a = *p.mlp_bwd;
    b.next_independent = first_bwd;  // B1 reads dZ and the saved H/U only (dZ of a stack's
                                     // inner layer is the next layer's dX: a real dependency)
    // B1: dH = dZ W2^T, all-reduce on dim 2 (conjugate of f4); dU = dH * GeLU'(U); || dW2, db2
    if (!b.stage(2, a.dz, hc, a.w2, hc, false, F1, nullptr, a.ws_dh, EPI_DGELU,
                 [&](EpiParams& ep, int64_t, int64_t) {
                   ep.aux = aux(a.u);
                   ep.ldaux = F1;
                 },
                 [&](int, int64_t r0, int64_t n) {
                   return EwList{E::ewd(EW_DGELU, mrows(a.ws_dh, r0, F1), rows(a.u, r0, F1), n, F1)};
                 },
                 [&]() { return b.dw(a.h_act, F1, a.dz, hc, a.dw2, a.db2); }))
      return fail();
    // B3: dX1 = dU W1^T, all-reduce on dim 1 (conjugate of f3); dX1 += dZ; || dW1, db1
    if (!b.stage(1, a.ws_dh, F1, a.w1, F1, false, hc, nullptr, a.dx, EPI_RESID,
                 [&](EpiParams& ep, int64_t, int64_t) {
                   ep.aux = aux(a.dz);
                   ep.ldaux = hc;
                 },
                 [&](int, int64_t r0, int64_t n) {
                   return EwList{E::ewd(EW_ADD, mrows(a.dx, r0, hc), rows(a.dz, r0, hc), n, hc)};
                 },
                 [&]() { return b.dw(a.x, hc, a.ws_dh, F1, a.dw1, a.db1); }))
      return fail();
  }
  if (!fwd && p.attn_bwd) {
    const atp_attn_bwd_args& a = *p.attn_bwd;
    // B4/B5: dctx = dY Wo^T, all-reduce on dim 2 (conjugate of f2); dQKV = expand(dctx); || dWo, dbo
    if (!b.stage(2, a.dy, hc, a.wo, hc, false, h1, nullptr, a.ws_dctx, EPI_BF16, no_fuse,
                 [&](int, int64_t r0, int64_t n) {
                   return EwList{E::ewd(EW_CORE_BWD, mrows(a.ws_dqkv, r0, q1), rows(a.ws_dctx, r0, h1), n, h1, hl)};
                 },
                 [&]() {
                   if (rv.d2 == 1) b.ew(E::ewd(EW_CORE_BWD, a.ws_dqkv, a.ws_dctx, T, h1, hl), 0);
                   return b.dw(a.ctx, h1, a.dy, hc, a.dwo, a.dbo);
                 }))
      return fail();
    // B6: dX = dQKV Wqkv^T, all-reduce on dim 1 (conjugate of f1); dX += dY; || dWqkv, dbqkv
    if (!b.stage(1, a.ws_dqkv, q1, a.wqkv, q1, false, hc, nullptr, a.dx, EPI_RESID,
                 [&](EpiParams& ep, int64_t, int64_t) {
                   ep.aux = aux(a.dy);
                   ep.ldaux = hc;
                 },
                 [&](int, int64_t r0, int64_t n) {
                   return EwList{E::ewd(EW_ADD, mrows(a.dx, r0, hc), rows(a.dy, r0, hc), n, hc)};
                 },
                 [&]() { return b.dw(a.x, hc, a.ws_dqkv, q1, a.dwqkv, a.dbqkv); }))
      return fail();
  }
  return true;
}

// A stack of n layers as ONE chunk pipeline (SURVEY §8(d) L_bench): forward
// layer 0..n-1, then backward n-1..0.  Layer l+1's first GEMM waits only for
// layer l's last stage (its chunk pipeline: per-chunk events / gates), so the
// last all-reduce of a layer overlaps the next layer's first GEMM (Fig. 7,
// P:328) instead of draining at a call boundary.
int build_layer_stack(const RankView& rv, const LayerParts* parts, int n_layers, int64_t T, int64_t h, int64_t F,
                      int64_t heads, int chunks, int dtype, Sched& out) {
  Builder b(rv, T, chunks, dtype);
  for (int l = 0; l < n_layers; ++l)
    if (!emit_layer(b, rv, parts[l], true, false, T, h, F, heads)) {
      set_error(b.err);
      return 2;
    }
  for (int l = n_layers - 1; l >= 0; --l)
    if (!emit_layer(b, rv, parts[l], false, l == n_layers - 1, T, h, F, heads)) {
      set_error(b.err);
      return 2;
    }
  b.flush();
  out = std::move(b.s);
  return 0;
}

int build_layer(const RankView& rv, const LayerParts& p, int64_t T, int64_t h, int64_t F, int64_t heads,
                int chunks, int dtype, Sched& out) {
  return build_layer_stack(rv, &p, 1, T, h, F, heads, chunks, dtype, out);
}


// ---------------------------------------------------------------- full GPT layer
namespace {

// Per-rank workspace of the full layer (bytes, 256-aligned pieces).
struct GptWs {
  size_t part, packed, ctxb, dctxp, dctxl, dqkvl, dqkvb, dqkv, dh, dbn, dy1, da, st1, st2, bs1, bs2, lnws, attn, total;
  size_t attn_bytes = 0;
  GptWs(int d1, int d2, int64_t T, int64_t h, int64_t F, int64_t heads, int64_t seq, int chunks) {
    (void)seq;
    const int64_t hc = h / d2, h1 = h / d1, q1 = 3 * h / d1, F1 = F / d1, ql = q1 / d2, cl = h1 / d2;
    const int64_t hl = heads / (d1 * d2), Mc = T / chunks;
    size_t off = 0;
    auto take = [&](size_t bytes) {
      const size_t o = off;
      off += (bytes + 255) & ~static_cast<size_t>(255);
      return o;
    };
    part = take(T * q1 * 2);
    packed = take(T * q1 * 2);
    ctxb = take(T * h1 * 2);
    dctxp = take(T * h1 * 2);
    dctxl = take(T * cl * 2);
    dqkvl = take(T * ql * 2);
    dqkvb = take(T * q1 * 2);
    dqkv = take(T * q1 * 2);
    dh = take(T * F1 * 2);
    dbn = take(T * hc * 2);
    dy1 = take(T * hc * 2);
    da = take(T * hc * 2);
    st1 = take(T * 8);
    st2 = take(T * 8);
    bs1 = take(T * 8);
    bs2 = take(T * 8);
    lnws = take(ln_param_workspace_bytes(hc));
    // backward scratch, also the forward's split-KV scratch on small grids
    attn = take(std::max(attn_workspace_bytes(Mc, static_cast<int>(hl)),
                         attn_fwd_split_bytes(Mc, seq, static_cast<int>(hl))));
    attn_bytes = std::max(attn_workspace_bytes(Mc, static_cast<int>(hl)),
                          attn_fwd_split_bytes(Mc, seq, static_cast<int>(hl)));
    total = off;
  }
};

}  // namespace

size_t gpt_workspace_bytes(int d1, int d2, int64_t T, int64_t h, int64_t F, int64_t heads, int64_t seq, int chunks) {
  return GptWs(d1, d2, T, h, F, heads, seq, chunks).total;
}

// Stages breadth-first over chunks (Fig. 7; reading G14): a chunk's op
// on the compute stream waits only for that chunk's previous collective; the
// elementwise step that follows a collective is deferred into the next
// stage's chunk prologue, so chunk k's collective overlaps the compute of the
// chunks before it.  dW GEMMs run on all T rows after their stage's chunks.
int build_gpt_layer(const RankView& rv, const atp_gpt_args& a, int64_t T, int64_t h, int64_t F, int64_t heads,
                    int64_t seq, int chunks, int causal, char* ws, Sched& out) {
  Builder b(rv, T, chunks, 0);
  const int d1 = rv.d1, d2 = rv.d2;
  const int64_t hc = h / d2, h1 = h / d1, q1 = 3 * h / d1, F1 = F / d1, ql = q1 / d2, cl = h1 / d2;
  const int hl = static_cast<int>(heads / (d1 * d2));
  const int64_t Mc = T / chunks;
  const GptWs L(d1, d2, T, h, F, heads, seq, chunks);
  auto W = [&](size_t off) { return static_cast<void*>(ws + off); };
  auto R = [&](const void* base, int k, int64_t w, int esz = 2) {  // chunk k's rows of a [T, w] buffer
    return static_cast<void*>(static_cast<char*>(const_cast<void*>(base)) + static_cast<int64_t>(k) * Mc * w * esz);
  };
  using E = Builder;
  auto fail = [&]() {
    set_error(b.err);
    return 2;
  };
  // compute-stream op of chunk k after its prologue (pending wait + deferred steps)
  auto gemm_k = [&](int k, const void* A, int64_t lda, const void* Wt, int64_t ldw, bool b_mn, int64_t N, int64_t K,
                    void* C, const void* bias, int epi, const void* aux, void* C2) {
    b.gate_slot = -1;  // custom ops in between: the next stage must not gate on older chunk gates
    const int w = b.prologue(k);
    EpiParams ep;
    ep.C = C;
    ep.ldc = N;
    ep.bias = bias;
    ep.aux = aux;
    ep.ldaux = N;
    ep.C2 = C2;
    ep.ldc2 = N;
    return b.gemm(A, lda, false, Wt, ldw, b_mn, Mc, N, K, epi, ep, {w}, -1) != nullptr;
  };
  auto ew_k = [&](int k, const EwDesc& e) {
    b.gate_slot = -1;
    const int w = b.prologue(k);
    b.ew(e, 0, w);
  };
  // collective of chunk k on the communication stream after the last compute op;
  // `post` runs in chunk k's next prologue
  auto coll_k = [&](int k, int dim, int coll, void* ptr, void* outp, int64_t count, int dtype, const EwList& post) {
    const int e = b.ev();
    b.s.ops.back().record = e;
    Op& o = b.push(OP_AR, 1);
    o.ar_dim = dim;
    o.coll = coll;
    o.ar_ptr = ptr;
    o.ar_out = outp;
    o.ar_count = count;
    o.ar_dtype = dtype;
    Builder::add_wait(o, e);
    const int r = b.ev();
    o.record = r;
    b.pend[k] = r;
    for (const EwDesc& d : post) b.def[k].push_back(d);
  };
  auto ln_stats = [&](const void* x, int64_t rows, float* st) {
    EwDesc e = E::ewd(EW_LN_STATS, nullptr, x, rows, hc);
    e.out2 = st;
    return e;
  };
  auto ln_apply = [&](const void* x, const void* g, const void* be, float* st, float* sv, void* y, int64_t rows) {
    EwDesc e = E::ewd(EW_LN_APPLY, y, x, rows, hc);
    e.b = g;
    e.c = be;
    e.out2 = st;
    e.ws = sv;
    e.n_total = h;
    return e;
  };
  auto ln_bstats = [&](const void* dy, const void* x, const void* g, float* sv, float* bs, int64_t rows) {
    EwDesc e = E::ewd(EW_LN_BWD_STATS, nullptr, dy, rows, hc);
    e.b = x;
    e.c = g;
    e.ws = sv;
    e.out2 = bs;
    return e;
  };
  auto ln_bapply = [&](const void* dy, const void* x, const void* g, float* sv, float* bs, const void* res, void* o,
                       int64_t rows) {
    EwDesc e = E::ewd(EW_LN_BWD_APPLY, o, dy, rows, hc);
    e.b = x;
    e.c = g;
    e.ws = sv;
    e.out2 = bs;
    e.res = res;
    e.n_total = h;
    return e;
  };
  auto ln_params = [&](const void* dy, const void* x, float* sv, float* dg, float* dbe) {
    EwDesc e = E::ewd(EW_LN_PARAM_GRAD, dg, dy, T, hc);
    e.b = x;
    e.ws = sv;
    e.res_out = dbe;
    e.out2 = W(L.lnws);
    b.ew(e, aux_colsum() ? 2 : 0, b.mark_compute());
  };
  // LayerNorm of every chunk: row statistics, dim-2 all-reduce (G33), apply (deferred)
  auto layernorm = [&](const void* x, const void* g, const void* be, size_t st_off, float* sv, void* y) {
    for (int k = 0; k < chunks; ++k) {
      if (d2 == 1) {  // the whole row is local: statistics + apply in one kernel
        EwDesc e = ln_apply(R(x, k, hc), g, be, nullptr, static_cast<float*>(R(sv, k, 2, 4)), R(y, k, hc), Mc);
        e.kind = EW_LN_FWD;
        ew_k(k, e);
        continue;
      }
      float* st = static_cast<float*>(R(W(st_off), k, 2, 4));
      ew_k(k, ln_stats(R(x, k, hc), Mc, st));
      const EwDesc ap = ln_apply(R(x, k, hc), g, be, st, static_cast<float*>(R(sv, k, 2, 4)), R(y, k, hc), Mc);
      if (d2 > 1)
        coll_k(k, 2, 0, st, nullptr, 2 * Mc, 1, {ap});
      else
        b.def[k].push_back(ap);
    }
  };
  auto ln_backward = [&](const void* dy, const void* x, const void* g, float* sv, size_t bs_off, const void* res,
                         void* o) {
    for (int k = 0; k < chunks; ++k) {
      float* bs = static_cast<float*>(R(W(bs_off), k, 2, 4));
      float* svk = static_cast<float*>(R(sv, k, 2, 4));
      if (d2 == 1) {  // statistics + apply in one kernel
        EwDesc e = ln_bapply(R(dy, k, hc), R(x, k, hc), g, svk, nullptr, R(res, k, hc), R(o, k, hc), Mc);
        e.kind = EW_LN_BWD;
        ew_k(k, e);
        continue;
      }
      ew_k(k, ln_bstats(R(dy, k, hc), R(x, k, hc), g, svk, bs, Mc));
      const EwDesc ap = ln_bapply(R(dy, k, hc), R(x, k, hc), g, svk, bs, R(res, k, hc), R(o, k, hc), Mc);
      if (d2 > 1)
        coll_k(k, 2, 0, bs, nullptr, 2 * Mc, 1, {ap});
      else
        b.def[k].push_back(ap);
    }
  };
  auto attn_desc = [&](int kind, int k) {
    EwDesc e;
    e.kind = kind;
    e.rows = Mc;
    e.heads = hl;
    e.seq = static_cast<int>(seq);
    e.causal = causal;
    e.out2 = R(a.lse, k, hl, 4);  // per-chunk [hl][Mc] block
    return e;
  };
  void* ctx_loc = d2 > 1 ? a.ctx_loc : a.ctx;
  const bool c1 = (d1 == 1), c2 = (d2 == 1);
  const void* bqkv_here = rv.i2 == 0 ? a.bqkv : nullptr;  // added once before the dim-2 reduction (G16)

  // ================= forward
  layernorm(a.x, a.g1, a.be1, L.st1, a.sv1, a.a);
  for (int k = 0; k < chunks; ++k) {  // QKV column-first; reduce-scatter of the head blocks on dim 2 (f1)
    void* dst = c2 ? R(a.qkv, k, ql) : R(W(L.part), k, q1);
    if (!gemm_k(k, R(a.a, k, hc), hc, a.wqkv, q1, true, q1, hc, dst, bqkv_here, EPI_BF16, nullptr, nullptr)) return fail();
    if (!c2) {
      EwDesc pk = E::ewd(EW_PACK, R(W(L.packed), k, q1), dst, Mc, q1);
      pk.p = d2;
      b.ew(pk, 0);
      coll_k(k, 2, 1, R(W(L.packed), k, q1), R(a.qkv, k, ql), Mc * ql, 0, {});
    }
  }
  for (int k = 0; k < chunks; ++k) {  // attention core on the local heads; all-gather ctx on dim 2 (f1 conjugate)
    EwDesc at = attn_desc(EW_ATTN_FWD, k);
    at.a = R(a.qkv, k, ql);
    at.lda = ql;
    at.out = R(ctx_loc, k, cl);
    at.ldo = cl;
    at.ws = W(L.attn);  // split-KV scratch (the chunks' forwards run in stream order, before any backward)
    at.n_total = static_cast<int64_t>(L.attn_bytes);
    ew_k(k, at);
    if (!c2) {
      EwDesc un = E::ewd(EW_UNPACK, R(a.ctx, k, h1), R(W(L.ctxb), k, h1), Mc, h1);
      un.p = d2;
      coll_k(k, 2, 2, R(ctx_loc, k, cl), R(W(L.ctxb), k, h1), Mc * cl, 0, {un});
    }
  }
  // Out row-first, all-reduce on dim 1 (f2), residual Y1 = X + .  (Builder::stage: one
  // signalled GEMM over all T rows when chunked and communicating, §6)
  if (!b.stage(1, a.ctx, h1, a.wo, hc, true, hc, a.bo, a.y1, EPI_RESID,
               [&](EpiParams& ep, int64_t, int64_t) {
                 ep.aux = a.x;
                 ep.ldaux = hc;
               },
               [&](int, int64_t r0, int64_t n) {
                 return EwList{E::ewd(EW_ADD, mptr(a.y1, r0 * hc), cptr(a.x, r0 * hc), n, hc)};
               },
               [] { return true; }))
    return fail();
  layernorm(a.y1, a.g2, a.be2, L.st2, a.sv2, a.bn);
  // FC1 column-first, all-reduce on dim 2 (f3), GeLU
  if (!b.stage(2, a.bn, hc, a.w1, F1, true, F1, a.b1, a.u, EPI_BIAS_GELU,
               [&](EpiParams& ep, int64_t, int64_t) {
                 ep.C2 = a.h;
                 ep.ldc2 = F1;
               },
               [&](int, int64_t r0, int64_t n) {
                 return EwList{E::ewd(EW_GELU, mptr(a.h, r0 * F1), cptr(a.u, r0 * F1), n, F1)};
               },
               [] { return true; }))
    return fail();
  // FC2 row-first, all-reduce on dim 1 (f4), residual Z = Y1 + .
  if (!b.stage(1, a.h, F1, a.w2, hc, true, hc, a.b2, a.z, EPI_RESID,
               [&](EpiParams& ep, int64_t, int64_t) {
                 ep.aux = a.y1;
                 ep.ldaux = hc;
               },
               [&](int, int64_t r0, int64_t n) {
                 return EwList{E::ewd(EW_ADD, mptr(a.z, r0 * hc), cptr(a.y1, r0 * hc), n, hc)};
               },
               [] { return true; }))
    return fail();

  // ================= backward
  void* dh = W(L.dh);
  b.next_independent = true;  // FC2-dX reads dZ and the saved U only
  // FC2-dX, all-reduce on dim 2, dGeLU; || dW2, db2
  if (!b.stage(2, a.dz, hc, a.w2, hc, false, F1, nullptr, dh, EPI_DGELU,
               [&](EpiParams& ep, int64_t, int64_t) {
                 ep.aux = a.u;
                 ep.ldaux = F1;
               },
               [&](int, int64_t r0, int64_t n) {
                 return EwList{E::ewd(EW_DGELU, mptr(dh, r0 * F1), cptr(a.u, r0 * F1), n, F1)};
               },
               [&]() { return b.dw(a.h, F1, a.dz, hc, a.dw2, a.db2); }))
    return fail();
  void* dbn = W(L.dbn);
  // FC1-dX, all-reduce on dim 1 (LayerNorm-2 backward follows); || dW1, db1
  if (!b.stage(1, dh, F1, a.w1, F1, false, hc, nullptr, dbn, EPI_BF16, [](EpiParams&, int64_t, int64_t) {},
               [](int, int64_t, int64_t) { return EwList{}; },
               [&]() { return b.dw(a.bn, hc, dh, F1, a.dw1, a.db1); }))
    return fail();
  void* dy1 = W(L.dy1);
  ln_backward(dbn, a.y1, a.g2, a.sv2, L.bs2, a.dz, dy1);  // dY1 = dZ + LN2'(dB)
  for (int k = 0; k < chunks; ++k) b.prologue(k);        // dY1 complete before dWo / LN2 params
  ln_params(dbn, a.y1, a.sv2, a.dg2, a.dbe2);
  void* dctxl = W(L.dctxl);
  for (int k = 0; k < chunks; ++k) {  // Out-dX, reduce-scatter of the head blocks on dim 2 (f2 conjugate)
    void* dst = c2 ? R(dctxl, k, cl) : R(W(L.dctxp), k, h1);
    if (!gemm_k(k, R(dy1, k, hc), hc, a.wo, hc, false, h1, hc, dst, nullptr, EPI_BF16, nullptr, nullptr)) return fail();
    if (!c2) {
      EwDesc pk = E::ewd(EW_PACK, R(W(L.packed), k, h1), dst, Mc, h1);
      pk.p = d2;
      b.ew(pk, 0);
      coll_k(k, 2, 1, R(W(L.packed), k, h1), R(dctxl, k, cl), Mc * cl, 0, {});
    }
  }
  if (!b.dw(a.ctx, h1, dy1, hc, a.dwo, a.dbo)) return fail();
  void* dqkv = W(L.dqkv);
  for (int k = 0; k < chunks; ++k) {  // attention backward on the local heads; all-gather dQKV on dim 2 (f1)
    EwDesc at = attn_desc(EW_ATTN_BWD, k);
    at.a = R(a.qkv, k, ql);
    at.lda = ql;
    at.b = R(ctx_loc, k, cl);
    at.ldb = cl;
    at.res = R(dctxl, k, cl);
    at.ldres = cl;
    at.out = c2 ? R(dqkv, k, q1) : R(W(L.dqkvl), k, ql);
    at.ldo = c2 ? q1 : ql;
    at.ws = W(L.attn);
    ew_k(k, at);
    if (!c2) {
      EwDesc un = E::ewd(EW_UNPACK, R(dqkv, k, q1), R(W(L.dqkvb), k, q1), Mc, q1);
      un.p = d2;
      coll_k(k, 2, 2, R(W(L.dqkvl), k, ql), R(W(L.dqkvb), k, q1), Mc * ql, 0, {un});
    }
  }
  void* da = W(L.da);
  // QKV-dX, all-reduce on dim 1 (LayerNorm-1 backward follows); || dWqkv, dbqkv
  if (!b.stage(1, dqkv, q1, a.wqkv, q1, false, hc, nullptr, da, EPI_BF16, [](EpiParams&, int64_t, int64_t) {},
               [](int, int64_t, int64_t) { return EwList{}; },
               [&]() { return b.dw(a.a, hc, dqkv, q1, a.dwqkv, a.dbqkv); }))
    return fail();
  ln_backward(da, a.x, a.g1, a.sv1, L.bs1, dy1, a.dx);  // dX = dY1 + LN1'(dA)
  for (int k = 0; k < chunks; ++k) b.prologue(k);
  ln_params(da, a.x, a.sv1, a.dg1, a.dbe1);
  b.flush();
  out = std::move(b.s);
  return 0;
}

}  // namespace atp
