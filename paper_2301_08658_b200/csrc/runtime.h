// Host runtime of libatp: mesh state, the op-list schedule and its executors.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <string>
#include <vector>

#include "atp_internal.h"
#include "elementwise.h"
#include "fused_ar.h"

struct atp_mesh;

namespace atp {

void set_error(const std::string& msg);

enum OpKind : int { OP_GEMM = 0, OP_EW = 1, OP_AR = 2, OP_WAITSIG = 3, OP_FUSED_AR = 4, OP_SIGNAL = 5 };

// kSigSlots (fused_ar.h): per-rank chunk-completion counters
constexpr int kMaxChunks = 16;   // chunk count limit (bounds the waits of one op)

// One enqueue on one of a rank's two streams.  `waits` are schedule-local
// event ids the op's stream waits on first; `record` is recorded after it.
struct Op {
  OpKind kind = OP_GEMM;
  int stream = 0;  // 0 = compute (caller's stream), 1 = communication, 2 = auxiliary
  int waits[kMaxChunks] = {};
  int n_waits = 0;
  int record = -1;
  GemmDesc g;
  EwDesc e;
  int ar_dim = 0;  // mesh dimension of the grouped collective (1 or 2)
  // OP_AR collective: 0 all-reduce (in place on ar_ptr, ar_count elements),
  // 1 reduce-scatter (ar_ptr [p][ar_count] -> ar_out [ar_count], member j keeps block j),
  // 2 all-gather (ar_ptr [ar_count] -> ar_out [p][ar_count], blocks in member order)
  int coll = 0;
  void* ar_ptr = nullptr;
  void* ar_out = nullptr;
  int64_t ar_count = 0;
  int ar_dtype = 0;      // 0 = bf16, 1 = fp32
  // OP_WAITSIG: the stream waits until counter `sig_slot` has grown by
  // `sig_inc` since the previous wait on that slot (cyclic >=).
  // OP_SIGNAL: the stream publishes gate `sig_slot` = the call's epoch.
  // OP_GEMM with g.gate: gate_slot0 = first slot of its gates (target filled in
  // at enqueue time from the published totals).
  int sig_slot = 0;
  uint32_t sig_inc = 0;
  int gate_slot0 = -1;
  // OP_FUSED_AR: static part of the fused all-reduce (targets and peer
  // pointers are filled in by the executor); ar_dim names the group.
  FusedArArgs far;
};

struct Sched {
  std::vector<Op> ops;
  int n_events = 0;
};

struct RankView {
  int d1 = 1, d2 = 1, i1 = 0, i2 = 0;
  int gemm_ctas = 0;
  uint32_t* sig_buf = nullptr;  // this rank's chunk-completion counters (device)
  bool signalled = true;        // use signalled stages when possible
  char* sym_base = nullptr;     // fused all-reduce: this rank's peer-visible buffer
  size_t sym_part_bytes = 0;    //   capacity of each of its two partial-sum regions
  char* peers[2][16] = {};      //   the dim-1 / dim-2 group members' buffers (fused GEMM push targets)
  int me_in[2] = {0, 0};        //   this rank's index in its dim-1 / dim-2 group
  bool gate_ok = false;         // chunk-gated GEMMs allowed (GEMM CTA cap leaves SMs free)
};

struct RankState {
  cudaStream_t comm = nullptr;
  cudaStream_t compute = nullptr;  // virtual mesh only (one per virtual rank)
  cudaStream_t aux = nullptr;      // off-critical-path work (bias-gradient column sums)
  std::vector<cudaEvent_t> ev;
  cudaEvent_t arrive = nullptr, done = nullptr, join = nullptr;
  uint32_t* sig_buf = nullptr;       // device counters [kSigSlots]
  bool sig_owned = true;             // false once moved into the symmetric buffer
  std::vector<uint32_t> sig_total;   // host mirror of the values the counters reach
  uint32_t epoch = 0;                // calls executed (chunk gates hold the epoch)
  // fused all-reduce ("symmetric" buffer: partials [part_bytes] + counters
  // tile[kSigSlots] ready[kSigSlots] done[kSigSlots]); peers per mesh dim
  char* sym_base = nullptr;
  size_t sym_part_bytes = 0;
  char* peers[2][16] = {};  // [dim-1][member index] -> member's sym_base
  int me_in[2] = {0, 0};
  std::vector<char*> ipc_opened;
  std::vector<uint32_t> ready_total, done_total;
};

}  // namespace atp

namespace atp {
struct ProfRec {
  cudaEvent_t a = nullptr, b = nullptr;
  int cls = 0;
  int stream = 0;  // 0 compute, 1 communication, 2 auxiliary
  int kind = 0;    // OpKind
  int sub = 0;     // GEMM epilogue kind / elementwise kind / collective kind
  double flops = 0, bytes = 0;
};
}  // namespace atp

struct atp_mesh {
  int d1 = 1, d2 = 1;
  bool comm_enabled = true;
  bool local_only = false;  // atp_mesh_init_local: no communicators
  bool comms_borrowed = false;  // atp_mesh_init_from_comms: dim1/dim2 belong to the caller, no world
  bool signalled = true;    // signalled stages (ATP_SIGNALLED=0 disables, for A/B runs)
  bool gated = false;       // chunk-gated GEMMs (atp_mesh_set_gating; ATP_GATED=1 initial value)
  bool profiling = false;
  void* capture_stream = nullptr;  // atp_graph_begin .. atp_graph_end: the stream being captured
  uint64_t capture_launch0 = 0;    // libatp launch count when the capture began
  std::vector<atp::ProfRec> prof;  // event pool; the first prof_used are live
  size_t prof_used = 0;
  bool is_virtual = false;
  int rank = 0, i1 = 0, i2 = 0;
  int device = 0;
  int gemm_ctas = 0;
  ncclComm_t world = nullptr, dim1 = nullptr, dim2 = nullptr;
  std::vector<atp::RankState> rs;  // 1 (distributed) or d1*d2 (virtual)
  cudaEvent_t ev_start = nullptr;
};

namespace atp {

RankView rank_view(const atp_mesh* m, int r);
// Run one schedule per rank (size 1 for a distributed mesh) on `stream`.
int execute(atp_mesh* m, std::vector<Sched>& per_rank, cudaStream_t stream);
void count_launch(uint64_t n);
uint64_t launch_count();
void op_cost(const Op& op, int p, int* cls, double* flops, double* bytes);
bool stream_wait_available();
int enable_fused_ar(atp_mesh* m, size_t part_bytes);
int debug_counters(atp_mesh* m, int rank, uint32_t* out, int n);
constexpr int kFusedCtas = 32;  // CTAs of one fused all-reduce kernel: 2 per SM on the 16 SMs the GEMM cap leaves
int fused_ctas();                // kFusedCtas, or ATP_FUSED_CTAS (SM-budget A/B runs)

}  // namespace atp
