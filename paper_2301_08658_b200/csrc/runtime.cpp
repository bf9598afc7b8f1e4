// Mesh lifetime and the two schedule executors.
//
// Distributed mesh (one process per GPU): the schedule's compute ops go
// on the caller's stream, its all-reduces on the mesh's communication stream
// as ncclAllReduce on the dim-1 / dim-2 communicator (grouped all-reduce,
// §3.2; communicators from ncclCommSplit, P:161 / P:270).  Cross-stream
// order is carried by CUDA events only; the host never synchronises.
//
// Virtual mesh (all d1*d2 ranks in one process on one GPU): the SAME per-rank
// schedules run in lockstep, op index by op index, each rank on its own
// compute and communication streams; a grouped all-reduce becomes one
// group_sum kernel per group on the group leader's communication stream,
// gated by events from every member (sum in ascending mesh coordinate, as the
// oracle does).  This lets a single B200 check the whole sharded pipeline —
// chunking, events, epilogues — for every mesh shape.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <atomic>
#include <cstdlib>
#include <mutex>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <string>

#include "runtime.h"

namespace atp {

namespace {
thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};
}  // namespace

void count_launch(uint64_t n) { g_launches += n; }

// cuStreamWaitValue32 from the driver (no link-time libcuda dependency).
static PFN_cuStreamWaitValue32_v11070 g_wait32 = nullptr;
static std::once_flag g_wait32_once;
bool stream_wait_available() {
  std::call_once(g_wait32_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_wait32 = reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(fn);
  });
  return g_wait32 != nullptr;
}

// Fill the dynamic part of a fused all-reduce and launch it (or, with the
// communication disabled, only account for the tile counter the GEMM bumped).
static cudaError_t launch_fused(atp_mesh* m, RankState& s, const Op& op, cudaStream_t st) {
  FusedArArgs a = op.far;
  if (m->is_virtual) {
    // Every rank's fused kernels share this one GPU and spin on one another's
    // progress: keep their CTAs together at one GPU's budget (kFusedCtas), or
    // they starve the CTA-pair GEMMs whose tiles they wait for (8 ranks x 32
    // spinning CTAs deadlocked every time once the streams ran truly
    // concurrently; with 2-8 CTAs per rank never: DESIGN.md §10).
    const int per = (kFusedCtas / (m->d1 * m->d2)) & ~1;
    a.n_ctas = std::max(2, std::min(a.n_ctas, per));
  }
  const int d = op.ar_dim - 1;
  a.p = op.ar_dim == 1 ? m->d1 : m->d2;
  a.me = s.me_in[d];
  for (int j = 0; j < a.p; ++j) a.peer_base[j] = s.peers[d][j];
  s.sig_total[a.sig_slot] += op.sig_inc;
  // a local dry-run mesh runs the kernel against its own buffer only (every
  // "peer" is itself): the per-rank cost of the fused step without NVLink.
  if (!m->comm_enabled && !m->local_only) return cudaSuccess;
  a.sig_target = s.sig_total[a.sig_slot];
  a.ready_target = (s.ready_total[a.sig_slot] += static_cast<uint32_t>(a.n_ctas));
  a.done_target = (s.done_total[a.sig_slot] += static_cast<uint32_t>(a.p * a.n_ctas));
  count_launch(2);  // phase A + phase B/C kernels
  return fused_ar_launch(a, st);
}

static PFN_cuStreamWriteValue32_v11070 g_write32 = nullptr;
static std::once_flag g_write32_once;
static bool stream_write_available() {
  std::call_once(g_write32_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_write32 = reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(fn);
  });
  return g_write32 != nullptr;
}

// Publish a chunk gate: gate = this call's epoch (the write follows all prior
// work of the stream and is preceded by a memory barrier).  Gates hold absolute
// epochs, not counts, so a slot's history (schedules with other chunk counts
// use other gate slots) never matters: a gate read >= epoch was written by
// this call.
static cudaError_t signal_gate(RankState& s, const Op& op, cudaStream_t st) {
  if (g_write32 == nullptr) return cudaErrorNotSupported;
  CUresult r = g_write32(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(s.sig_buf + op.sig_slot),
                         s.epoch, CU_STREAM_WRITE_VALUE_DEFAULT);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorUnknown;
}

static void fill_gate(RankState& s, Op& op) {
  if (op.kind == OP_GEMM && op.gate_slot0 >= 0) {
    op.g.gate = s.sig_buf + op.gate_slot0;
    op.g.gate_target = s.epoch;
  }
}

static cudaError_t wait_sig(RankState& s, const Op& op, cudaStream_t st) {
  s.sig_total[op.sig_slot] += op.sig_inc;
  CUresult r = g_wait32(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(s.sig_buf + op.sig_slot),
                        s.sig_total[op.sig_slot], CU_STREAM_WAIT_VALUE_GEQ);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorUnknown;
}
uint64_t launch_count() { return g_launches.load(); }
int fused_ctas() {
  static const int v = [] {
    const char* e = getenv("ATP_FUSED_CTAS");
    const int n = e ? atoi(e) : 0;
    return n > 0 ? (n + 1) / 2 * 2 : kFusedCtas;  // even: the kernels launch as 2-CTA clusters
  }();
  return v;
}

// Algorithmic cost of one op (class 0 = GEMM, 1 = elementwise, 2 = all-reduce).
void op_cost(const Op& op, int p, int* cls, double* flops, double* bytes) {
  *flops = 0;
  *bytes = 0;
  if (op.kind == OP_GEMM) {
    const double M = op.g.M, N = op.g.N, K = op.g.K;
    *cls = 0;
    *flops = 2.0 * M * N * K;
    double out = op.g.epi == EPI_F32 ? 4.0 : 2.0;
    double extra = (op.g.epi == EPI_RESID || op.g.epi == EPI_DGELU || op.g.epi == EPI_BIAS_GELU) ? 2.0 : 0.0;
    *bytes = 2.0 * (M * K + N * K) + M * N * (out + extra);
  } else if (op.kind == OP_EW && (op.e.kind == EW_ATTN_FWD || op.e.kind == EW_ATTN_BWD)) {
    // attention core: 4 d s_visible FLOPs per query row and head forward (QK^T and PV),
    // 2.5x that backward (5 products); causal rows see (s+1)/2 keys on average
    *cls = 3;
    const double s = op.e.seq, rows = static_cast<double>(op.e.rows), d = 128.0;
    const double keys = op.e.causal ? (s + 1.0) / 2.0 : s;
    const double f = 4.0 * d * keys * rows * op.e.heads;
    *flops = op.e.kind == EW_ATTN_FWD ? f : 2.5 * f;
    *bytes = (op.e.kind == EW_ATTN_FWD ? 8.0 : 20.0) * rows * op.e.heads * d;
  } else if (op.kind == OP_EW) {
    *cls = 1;
    const double n = static_cast<double>(op.e.rows) * op.e.cols;
    switch (op.e.kind) {
      case EW_GELU: *bytes = 4.0 * n; break;
      case EW_DGELU: case EW_ADD: *bytes = 6.0 * n; break;
      case EW_CORE_FWD: case EW_CORE_BWD: *bytes = 8.0 * n; break;
      case EW_COLSUM: *bytes = 2.0 * n + 4.0 * op.e.cols; break;
      case EW_LN_STATS: case EW_PACK: case EW_UNPACK: *bytes = (op.e.kind == EW_LN_STATS ? 2.0 : 4.0) * n; break;
      case EW_LN_APPLY: case EW_LN_BWD_STATS: *bytes = 4.0 * n; break;
      case EW_LN_BWD_APPLY: *bytes = 8.0 * n; break;
      case EW_LN_FWD: *bytes = 4.0 * n; break;   // x read once, y written
      case EW_LN_BWD: *bytes = 8.0 * n; break;   // dy, x, res read once, out written
      case EW_LN_PARAM_GRAD: *bytes = 4.0 * n; break;
      default: break;
    }
  } else {
    *cls = 2;
    const double esz = op.ar_dtype == 1 ? 4.0 : 2.0;
    if (p <= 1) *bytes = 0.0;
    else if (op.coll == 0) *bytes = 2.0 * (p - 1) / p * op.ar_count * esz;
    else *bytes = (p - 1.0) * op.ar_count * esz;  // reduce-scatter / all-gather ring
  }
}

// Profiling: bracket an enqueue with timing events on its stream.
static ProfRec* prof_begin(atp_mesh* m, const Op& op, cudaStream_t st) {
  if (!m->profiling) return nullptr;
  if (m->prof_used == m->prof.size()) {
    ProfRec r;
    if (cudaEventCreate(&r.a) != cudaSuccess || cudaEventCreate(&r.b) != cudaSuccess) return nullptr;
    m->prof.push_back(r);
  }
  ProfRec* r = &m->prof[m->prof_used++];
  const int p = op.kind == OP_AR ? (op.ar_dim == 1 ? m->d1 : m->d2) : 1;
  op_cost(op, p, &r->cls, &r->flops, &r->bytes);
  r->stream = op.stream;
  r->kind = op.kind;
  r->sub = op.kind == OP_GEMM ? op.g.epi : (op.kind == OP_EW ? op.e.kind : op.coll);
  cudaEventRecord(r->a, st);
  return r;
}
static void prof_end(ProfRec* r, cudaStream_t st) {
  if (r) cudaEventRecord(r->b, st);
}

void set_error(const std::string& msg) { g_err = msg; }
const char* last_error() { return g_err.c_str(); }

RankView rank_view(const atp_mesh* m, int r) {
  RankView v;
  v.d1 = m->d1;
  v.d2 = m->d2;
  if (m->is_virtual) {
    v.i1 = r / m->d2;
    v.i2 = r % m->d2;
  } else {
    v.i1 = m->i1;
    v.i2 = m->i2;
  }
  v.gemm_ctas = m->gemm_ctas;
  v.sig_buf = m->rs[m->is_virtual ? r : 0].sig_buf;
  v.sym_base = m->rs[m->is_virtual ? r : 0].sym_base;
  v.sym_part_bytes = m->rs[m->is_virtual ? r : 0].sym_part_bytes;
  for (int d = 0; d < 2; ++d) {
    const RankState& s = m->rs[m->is_virtual ? r : 0];
    for (int j = 0; j < 16; ++j) v.peers[d][j] = s.peers[d][j];
    v.me_in[d] = s.me_in[d];
  }
  v.signalled = m->signalled && stream_wait_available();
  {
    // Opt-in (ATP_GATED=1).  A gated GEMM spins on SMs it holds: only allowed
    // when its CTA cap leaves SMs for the communication-stream kernels that
    // release the gates.  Off by default: with the collectives elided, gating
    // made the per-rank compute 5-15% slower (the elementwise tails run on the
    // SMs the cap leaves free while the GEMM waits), and its gain
    // (overlapping the all-reduce tail) cannot be measured on one GPU.
    const int n_ranks = static_cast<int>(m->rs.size());
    v.gate_ok = m->gated && v.signalled && stream_write_available() && m->gemm_ctas > 0 &&
                m->gemm_ctas * n_ranks <= num_sms() - 16;
  }
  return v;
}

static int cuda_fail(cudaError_t e, const char* what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return 3;  // ATP_ERR_CUDA
}

static int ensure_events(RankState& s, int n) {
  while (static_cast<int>(s.ev.size()) < n) {
    cudaEvent_t e;
    cudaError_t err = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    if (err != cudaSuccess) return cuda_fail(err, "cudaEventCreate");
    s.ev.push_back(e);
  }
  return 0;
}

// `prev_kernel`: the previous enqueue on this stream in this call was one of
// our kernels.  Only then may a GEMM use programmatic dependent launch (its
// one dependency is that kernel; see GemmDesc::pdl): no event wait, no gate
// spin, no chunk counters (which the per-call reset must precede), no profiling.
static cudaError_t launch_local(Op& op, cudaStream_t st, bool prev_kernel, bool profiling) {
  if (op.kind == OP_GEMM) {
    count_launch(1);
    // A signalled GEMM may use PDL too: it touches no global memory (nor its
    // chunk counters) before griddepcontrol.wait, and the per-call counter
    // reset is a memset, never the kernel right before it.
    op.g.pdl = prev_kernel && !profiling && op.n_waits == 0 && op.g.gate == nullptr;
    return gemm_launch(op.g, st);
  }
  count_launch(op.e.kind == EW_ATTN_BWD ? 3 : (op.e.kind == EW_LN_PARAM_GRAD ? 2 : 1));
  return ew_launch(op.e, st);
}

// One grouped NCCL collective of a distributed mesh.
static int nccl_coll(atp_mesh* m, const Op& op, cudaStream_t st) {
  ncclComm_t comm = op.ar_dim == 1 ? m->dim1 : m->dim2;
  const ncclDataType_t dt = op.ar_dtype == 1 ? ncclFloat32 : ncclBfloat16;
  const size_t n = static_cast<size_t>(op.ar_count);
  ncclResult_t nr;
  const char* what;
  if (op.coll == 1) {
    nr = ncclReduceScatter(op.ar_ptr, op.ar_out, n, dt, ncclSum, comm, st);
    what = "ncclReduceScatter: ";
  } else if (op.coll == 2) {
    nr = ncclAllGather(op.ar_ptr, op.ar_out, n, dt, comm, st);
    what = "ncclAllGather: ";
  } else {
    nr = ncclAllReduce(op.ar_ptr, op.ar_ptr, n, dt, ncclSum, comm, st);
    what = "ncclAllReduce: ";
  }
  if (nr != ncclSuccess) {
    set_error(std::string(what) + ncclGetErrorString(nr));
    return 4;
  }
  return 0;
}

static cudaError_t wait_all(const Op& op, RankState& s, cudaStream_t st) {
  for (int w = 0; w < op.n_waits; ++w) {
    cudaError_t e = cudaStreamWaitEvent(st, s.ev[op.waits[w]], 0);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

int execute(atp_mesh* m, std::vector<Sched>& sch, cudaStream_t stream) {
  const int n = static_cast<int>(sch.size());
  if (n != static_cast<int>(m->rs.size())) {
    set_error("internal: schedule count != rank count");
    return 1;
  }
  for (int r = 0; r < n; ++r) {
    if (sch[r].ops.size() != sch[0].ops.size()) {
      set_error("internal: rank schedules differ in length");
      return 1;
    }
    int rc = ensure_events(m->rs[r], sch[r].n_events);
    if (rc) return rc;
  }
  cudaError_t e = cudaSuccess;
  // Without peer-memory all-reduce, a rank's chunk counters and gates are read
  // only by its own streams, so every call starts from zeroed counters (one
  // memset, ordered after the previous call's join): each call is
  // self-contained, which is what makes a captured CUDA graph replayable.
  // Fused meshes keep cumulative counters (peers may still read them).
  for (int r = 0; r < n; ++r) {
    RankState& s = m->rs[r];
    if (s.sym_base != nullptr) {
      ++s.epoch;
      continue;
    }
    if ((e = cudaMemsetAsync(s.sig_buf, 0, kSigSlots * sizeof(uint32_t), stream)) != cudaSuccess)
      return cuda_fail(e, "counter reset");
    std::fill(s.sig_total.begin(), s.sig_total.end(), 0u);
    s.epoch = 1;
  }
  e = cudaEventRecord(m->ev_start, stream);
  if (e != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
  for (int r = 0; r < n; ++r) {
    cudaStreamWaitEvent(m->rs[r].comm, m->ev_start, 0);
    cudaStreamWaitEvent(m->rs[r].aux, m->ev_start, 0);
    if (m->is_virtual) cudaStreamWaitEvent(m->rs[r].compute, m->ev_start, 0);
  }

  if (!m->is_virtual) {
    RankState& s = m->rs[0];
    bool prevk[3] = {false, false, false};
    for (Op& op : sch[0].ops) {
      cudaStream_t st = op.stream == 1 ? s.comm : (op.stream == 2 ? s.aux : stream);
      if ((e = wait_all(op, s, st)) != cudaSuccess) return cuda_fail(e, "cudaStreamWaitEvent");
      fill_gate(s, op);
      if (op.kind == OP_SIGNAL) {
        if ((e = signal_gate(s, op, st)) != cudaSuccess) return cuda_fail(e, "cuStreamWriteValue32");
        if (op.record >= 0) cudaEventRecord(s.ev[op.record], st);
        prevk[op.stream] = false;
        continue;
      }
      if (op.kind == OP_WAITSIG) {
        if ((e = wait_sig(s, op, st)) != cudaSuccess) return cuda_fail(e, "cuStreamWaitValue32");
        if (op.record >= 0) cudaEventRecord(s.ev[op.record], st);
        prevk[op.stream] = false;
        continue;
      }
      ProfRec* pr = prof_begin(m, op, st);
      if (op.kind == OP_FUSED_AR) {
        if ((e = launch_fused(m, s, op, st)) != cudaSuccess) return cuda_fail(e, "fused all-reduce launch");
      } else if (op.kind == OP_AR) {
        if (m->comm_enabled) {
          const int rc = nccl_coll(m, op, st);
          if (rc) return rc;
        }
      } else if ((e = launch_local(op, st, prevk[op.stream] && op.n_waits == 0, m->profiling)) != cudaSuccess) {
        return cuda_fail(e, op.kind == OP_GEMM ? "gemm launch" : "elementwise launch");
      }
      prevk[op.stream] = op.kind == OP_GEMM || op.kind == OP_EW;
      prof_end(pr, st);
      if (op.record >= 0) cudaEventRecord(s.ev[op.record], st);
    }
    cudaEventRecord(s.join, s.comm);
    cudaStreamWaitEvent(stream, s.join, 0);
    cudaEventRecord(s.join, s.aux);
    cudaStreamWaitEvent(stream, s.join, 0);
    return 0;
  }

  // ---------------------------------------------------- virtual lockstep
  const size_t n_ops = sch[0].ops.size();
  for (size_t i = 0; i < n_ops; ++i) {
    const OpKind kind = sch[0].ops[i].kind;
    for (int r = 0; r < n; ++r) {
      if (sch[r].ops[i].kind != kind) {
        set_error("internal: rank schedules differ in structure");
        return 1;
      }
    }
    if (kind != OP_AR) {
      for (int r = 0; r < n; ++r) {
        Op& op = sch[r].ops[i];
        RankState& s = m->rs[r];
        cudaStream_t st = op.stream == 1 ? s.comm : (op.stream == 2 ? s.aux : s.compute);
        if ((e = wait_all(op, s, st)) != cudaSuccess) return cuda_fail(e, "cudaStreamWaitEvent");
        fill_gate(s, op);
        if (op.kind == OP_SIGNAL) {
          if ((e = signal_gate(s, op, st)) != cudaSuccess) return cuda_fail(e, "cuStreamWriteValue32");
          if (op.record >= 0) cudaEventRecord(s.ev[op.record], st);
          continue;
        }
        if (op.kind == OP_WAITSIG) {
          if ((e = wait_sig(s, op, st)) != cudaSuccess) return cuda_fail(e, "cuStreamWaitValue32");
          if (op.record >= 0) cudaEventRecord(s.ev[op.record], st);
          continue;
        }
        ProfRec* pr = prof_begin(m, op, st);
        if (op.kind == OP_FUSED_AR) {
          if ((e = launch_fused(m, s, op, st)) != cudaSuccess) return cuda_fail(e, "fused all-reduce launch");
        } else if ((e = launch_local(op, st, false, m->profiling)) != cudaSuccess) {  // virtual mesh: no PDL
          return cuda_fail(e, op.kind == OP_GEMM ? "gemm launch" : "elementwise launch");
        }
        prof_end(pr, st);
        if (op.record >= 0) cudaEventRecord(s.ev[op.record], st);
      }
      continue;
    }
    const int dim = sch[0].ops[i].ar_dim;
    for (int r = 0; r < n; ++r) {
      if ((e = wait_all(sch[r].ops[i], m->rs[r], m->rs[r].comm)) != cudaSuccess)
        return cuda_fail(e, "cudaStreamWaitEvent");
    }
    const int ngroups = dim == 1 ? m->d2 : m->d1;
    const int p = dim == 1 ? m->d1 : m->d2;
    if (p > kMaxGroup) {
      set_error("virtual mesh: group larger than 16");
      return 1;
    }
    for (int g = 0; g < ngroups; ++g) {
      int members[kMaxGroup];
      for (int j = 0; j < p; ++j) members[j] = dim == 1 ? (j * m->d2 + g) : (g * m->d2 + j);
      const int leader = members[0];
      GroupSumArgs ga;
      ga.p = p;
      for (int j = 0; j < p; ++j) {
        ga.buf[j] = sch[members[j]].ops[i].ar_ptr;
        if (j > 0) {
          cudaEventRecord(m->rs[members[j]].arrive, m->rs[members[j]].comm);
          cudaStreamWaitEvent(m->rs[leader].comm, m->rs[members[j]].arrive, 0);
        }
      }
      ProfRec* pr = prof_begin(m, sch[leader].ops[i], m->rs[leader].comm);
      const Op& lop = sch[leader].ops[i];
      const size_t esz = lop.ar_dtype == 1 ? 4 : 2;
      cudaStream_t ls = m->rs[leader].comm;
      if (m->comm_enabled && lop.coll == 2) {
        // all-gather: member i's block -> block i of every member's output
        for (int jo = 0; jo < p; ++jo)
          for (int ji = 0; ji < p; ++ji)
            if ((e = cudaMemcpyAsync(static_cast<char*>(sch[members[jo]].ops[i].ar_out) + ji * lop.ar_count * esz,
                                     sch[members[ji]].ops[i].ar_ptr, lop.ar_count * esz, cudaMemcpyDeviceToDevice,
                                     ls)) != cudaSuccess)
              return cuda_fail(e, "virtual all-gather copy");
      } else if (m->comm_enabled) {
        const int64_t n_sum = lop.coll == 1 ? lop.ar_count * p : lop.ar_count;
        if ((e = group_sum_launch(ga, n_sum, lop.ar_dtype, ls)) != cudaSuccess) return cuda_fail(e, "group_sum launch");
        count_launch(1);
        if (lop.coll == 1)  // reduce-scatter: member j keeps block j of the sum
          for (int j = 0; j < p; ++j)
            if ((e = cudaMemcpyAsync(sch[members[j]].ops[i].ar_out,
                                     static_cast<char*>(sch[members[j]].ops[i].ar_ptr) + j * lop.ar_count * esz,
                                     lop.ar_count * esz, cudaMemcpyDeviceToDevice, ls)) != cudaSuccess)
              return cuda_fail(e, "virtual reduce-scatter copy");
      }
      prof_end(pr, m->rs[leader].comm);
      cudaEventRecord(m->rs[leader].done, m->rs[leader].comm);
      for (int j = 1; j < p; ++j) cudaStreamWaitEvent(m->rs[members[j]].comm, m->rs[leader].done, 0);
    }
    for (int r = 0; r < n; ++r) {
      const Op& op = sch[r].ops[i];
      if (op.record >= 0) cudaEventRecord(m->rs[r].ev[op.record], m->rs[r].comm);
    }
  }
  for (int r = 0; r < n; ++r) {
    RankState& s = m->rs[r];
    cudaEventRecord(s.join, s.comm);
    cudaStreamWaitEvent(stream, s.join, 0);
    cudaEventRecord(s.join, s.compute);
    cudaStreamWaitEvent(stream, s.join, 0);
    cudaEventRecord(s.join, s.aux);
    cudaStreamWaitEvent(stream, s.join, 0);
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "virtual executor");
  return 0;
}

// ---------------------------------------------------------------- fused all-reduce setup
// Every rank gets one "symmetric" allocation: the partial-sum region followed by
// its counters (tile / ready / done).  The GEMM counters move into it so peers
// can read them.  Virtual mesh: peers are the other virtual ranks' allocations;
// distributed mesh: CUDA IPC handles all-gathered over the world communicator
// and opened for the members of this rank's dim-1 and dim-2 groups.
int debug_counters(atp_mesh* m, int rank, uint32_t* out, int n) {
  RankState& s = m->rs[m->is_virtual ? rank : 0];
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaMemcpyAsync(out, s.sig_buf, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  for (int i = 0; i < n && i < static_cast<int>(s.sig_total.size()); ++i) out[n + i] = s.sig_total[i];
  return e == cudaSuccess ? 0 : 3;
}

int enable_fused_ar(atp_mesh* m, size_t part_bytes) {
  // the peer tables (RankState::peers, FusedArArgs::peer_base) hold 16 members per group
  if (m->d1 > 16 || m->d2 > 16) {
    set_error("fused all-reduce: mesh dimensions above 16 are not supported (peer tables hold 16 members)");
    return 1;
  }
  part_bytes = (part_bytes + 255) & ~static_cast<size_t>(255);
  const size_t flag_bytes = 3 * static_cast<size_t>(kSigSlots) * sizeof(uint32_t);
  const int n_local = static_cast<int>(m->rs.size());
  for (int r = 0; r < n_local; ++r) {
    RankState& s = m->rs[r];
    if (s.sym_base != nullptr) {
      set_error("fused all-reduce already enabled on this mesh");
      return 1;
    }
    // two partial regions: consecutive fused stages alternate, so a stage's GEMM
    // never overwrites partial sums the previous stage's all-reduce still reads
    cudaError_t e = cudaMalloc(&s.sym_base, 2 * part_bytes + flag_bytes);
    if (e == cudaSuccess) e = cudaMemset(s.sym_base + 2 * part_bytes, 0, flag_bytes);
    if (e != cudaSuccess) return cuda_fail(e, "fused all-reduce buffer");
    s.sym_part_bytes = part_bytes;
    if (s.sig_owned) cudaFree(s.sig_buf);
    s.sig_buf = reinterpret_cast<uint32_t*>(s.sym_base + 2 * part_bytes);
    s.sig_owned = false;
    s.sig_total.assign(kSigSlots, 0u);
    s.ready_total.assign(kSigSlots, 0u);
    s.done_total.assign(kSigSlots, 0u);
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(e, "fused all-reduce setup");
  const int d1 = m->d1, d2 = m->d2;
  if (m->is_virtual) {
    for (int r = 0; r < n_local; ++r) {
      const int i1 = r / d2, i2 = r % d2;
      RankState& s = m->rs[r];
      for (int j = 0; j < d1; ++j) s.peers[0][j] = m->rs[j * d2 + i2].sym_base;
      for (int j = 0; j < d2; ++j) s.peers[1][j] = m->rs[i1 * d2 + j].sym_base;
      s.me_in[0] = i1;
      s.me_in[1] = i2;
    }
    return 0;
  }
  RankState& s = m->rs[0];
  const int n = d1 * d2;
  std::vector<cudaIpcMemHandle_t> all(n);
  if (!m->local_only && n > 1) {
    if (m->world == nullptr) {
      set_error("fused all-reduce: needs the world communicator (not available with borrowed communicators)");
      return 1;
    }
    cudaIpcMemHandle_t h;
    if ((e = cudaIpcGetMemHandle(&h, s.sym_base)) != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
    uint8_t* dbuf = nullptr;
    if ((e = cudaMalloc(&dbuf, sizeof(h) * (n + 1))) != cudaSuccess) return cuda_fail(e, "ipc exchange buffer");
    cudaMemcpy(dbuf, &h, sizeof(h), cudaMemcpyHostToDevice);
    ncclResult_t r = ncclAllGather(dbuf, dbuf + sizeof(h), sizeof(h), ncclUint8, m->world, s.comm);
    cudaStreamSynchronize(s.comm);
    if (r == ncclSuccess) cudaMemcpy(all.data(), dbuf + sizeof(h), sizeof(h) * n, cudaMemcpyDeviceToHost);
    cudaFree(dbuf);
    if (r != ncclSuccess) {
      set_error(std::string("ipc handle exchange: ") + ncclGetErrorString(r));
      return 4;
    }
  }
  auto open = [&](int rank) -> char* {
    if (rank == m->rank || m->local_only) return s.sym_base;
    void* p = nullptr;
    cudaError_t err = cudaIpcOpenMemHandle(&p, all[rank], cudaIpcMemLazyEnablePeerAccess);
    if (err != cudaSuccess) {
      cuda_fail(err, "cudaIpcOpenMemHandle");
      return nullptr;
    }
    s.ipc_opened.push_back(static_cast<char*>(p));
    return static_cast<char*>(p);
  };
  for (int j = 0; j < d1; ++j)
    if (!(s.peers[0][j] = open(j * d2 + m->i2))) return 3;
  for (int j = 0; j < d2; ++j)
    if (!(s.peers[1][j] = open(m->i1 * d2 + j))) return 3;
  s.me_in[0] = m->i1;
  s.me_in[1] = m->i2;
  return 0;
}

// ---------------------------------------------------------------- mesh lifetime
static int make_rank_state(RankState& s, bool with_compute) {
  int lo, hi;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  cudaError_t e = cudaStreamCreateWithPriority(&s.comm, cudaStreamNonBlocking, hi);
  if (e == cudaSuccess && with_compute) e = cudaStreamCreateWithFlags(&s.compute, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&s.aux, cudaStreamNonBlocking, lo);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s.arrive, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s.join, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaMalloc(&s.sig_buf, kSigSlots * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemset(s.sig_buf, 0, kSigSlots * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(e, "stream/event/counter create");
  s.sig_total.assign(kSigSlots, 0u);
  return 0;
}

static void free_rank_state(RankState& s) {
  for (cudaEvent_t ev : s.ev) cudaEventDestroy(ev);
  s.ev.clear();
  if (s.arrive) cudaEventDestroy(s.arrive);
  if (s.done) cudaEventDestroy(s.done);
  if (s.join) cudaEventDestroy(s.join);
  if (s.comm) cudaStreamDestroy(s.comm);
  if (s.compute) cudaStreamDestroy(s.compute);
  if (s.aux) cudaStreamDestroy(s.aux);
  if (s.sig_buf && s.sig_owned) cudaFree(s.sig_buf);
  for (char* p : s.ipc_opened) cudaIpcCloseMemHandle(p);
  if (s.sym_base) cudaFree(s.sym_base);
  s = RankState();
}

int mesh_create(int d1, int d2, int world_rank, const uint8_t* uid, int device, bool is_virtual,
                atp_mesh** out) {
  if (out == nullptr) {
    set_error("atp_mesh_init: out is NULL");
    return 1;
  }
  *out = nullptr;
  if (d1 < 1 || d2 < 1) {
    set_error("atp_mesh_init: d1 and d2 must be >= 1");
    return 1;
  }
  const int n = d1 * d2;
  if (!is_virtual && (world_rank < 0 || world_rank >= n)) {
    set_error("atp_mesh_init: world_rank out of range");
    return 1;
  }
  if (is_virtual && (d1 > kMaxGroup || d2 > kMaxGroup)) {
    set_error("atp_vmesh_init: mesh dimensions above 16 unsupported");
    return 1;
  }
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  atp_mesh* m = new atp_mesh();
  m->d1 = d1;
  m->d2 = d2;
  m->is_virtual = is_virtual;
  m->device = device;
  m->rank = is_virtual ? 0 : world_rank;
  {
    const char* e = getenv("ATP_SIGNALLED");
    m->signalled = !(e && e[0] == '0');
    const char* g = getenv("ATP_GATED");
    m->gated = g && g[0] == '1';
  }
  m->i1 = m->rank / d2;
  m->i2 = m->rank % d2;
  m->rs.resize(is_virtual ? n : 1);
  for (auto& s : m->rs) {
    int rc = make_rank_state(s, is_virtual);
    if (rc) {
      for (auto& t : m->rs) free_rank_state(t);
      delete m;
      return rc;
    }
  }
  cudaEventCreateWithFlags(&m->ev_start, cudaEventDisableTiming);
  if (!is_virtual && uid == nullptr) {
    m->comm_enabled = false;  // local dry-run rank: no communicators, collectives elided
    m->local_only = true;
  } else if (!is_virtual) {
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&m->world, n, id, world_rank);
    // dim-1 group: the d1 ranks sharing i2 (color i2, ordered by i1); dim-2: sharing i1.
    // The dim communicators carry the data-path all-reduces, which overlap the
    // persistent GEMMs: bound NCCL's SM footprint to the SMs the GEMM CTA cap
    // leaves (bench: 132 of 148 -> 16; ATP_NCCL_MAX_CTAS overrides, 0 = NCCL's
    // default), so the two never compete for the same SMs.
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    {
      const char* e = getenv("ATP_NCCL_MAX_CTAS");
      const int mx = e ? atoi(e) : 16;
      if (mx > 0) cfg.maxCTAs = mx;
    }
    if (r == ncclSuccess) r = ncclCommSplit(m->world, m->i2, m->i1, &m->dim1, &cfg);
    if (r == ncclSuccess) r = ncclCommSplit(m->world, m->i1, m->i2, &m->dim2, &cfg);
    if (r != ncclSuccess) {
      set_error(std::string("NCCL mesh init: ") + ncclGetErrorString(r));
      if (m->dim1) ncclCommDestroy(m->dim1);
      if (m->world) ncclCommDestroy(m->world);
      for (auto& t : m->rs) free_rank_state(t);
      delete m;
      return 4;
    }
  }
  *out = m;
  return 0;
}

int mesh_destroy(atp_mesh* m) {
  if (m == nullptr) return 0;
  cudaSetDevice(m->device);
  for (auto& s : m->rs) {
    if (s.comm) cudaStreamSynchronize(s.comm);
    if (s.compute) cudaStreamSynchronize(s.compute);
    if (s.aux) cudaStreamSynchronize(s.aux);
  }
  if (!m->comms_borrowed) {
    if (m->dim2) ncclCommDestroy(m->dim2);
    if (m->dim1) ncclCommDestroy(m->dim1);
  }
  if (m->world) ncclCommDestroy(m->world);
  for (auto& s : m->rs) free_rank_state(s);
  for (auto& r : m->prof) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  if (m->ev_start) cudaEventDestroy(m->ev_start);
  delete m;
  return 0;
}

}  // namespace atp
