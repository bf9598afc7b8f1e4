// extern "C" entry points of libatp (declared and documented in include/atp.h).
// Every entry validates its arguments before anything is enqueued.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>
#include <string>
#include <vector>

#include "../../include/atp.h"
#include "attention.h"
#include "schedule.h"

using atp::Sched;

namespace {

atp_status fail(atp_status s, const std::string& msg) {
  atp::set_error(msg);
  return s;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

int n_ranks(const atp_mesh* m) { return static_cast<int>(m->rs.size()); }

template <class Build>
atp_status run(atp_mesh* m, void* stream, Build build) {
  const int n = n_ranks(m);
  std::vector<Sched> s(n);
  for (int r = 0; r < n; ++r) {
    int rc = build(atp::rank_view(m, r), r, s[r]);
    if (rc) return static_cast<atp_status>(rc);
  }
  cudaSetDevice(m->device);
  return static_cast<atp_status>(atp::execute(m, s, as_stream(stream)));
}

atp_status check_mesh(const atp_mesh* m, const void* args) {
  if (m == nullptr) return fail(ATP_ERR_INVALID, "mesh is NULL");
  if (args == nullptr) return fail(ATP_ERR_INVALID, "args is NULL");
  return ATP_OK;
}

bool w8(int64_t x) { return x > 0 && x % 8 == 0; }

}  // namespace

extern "C" {

const char* atp_last_error(void) { return atp::last_error(); }
const char* atp_version(void) { return ATP_VERSION; }

// ---------------------------------------------------------------- mesh
atp_status atp_get_unique_id(uint8_t uid_out[128]) {
  if (uid_out == nullptr) return fail(ATP_ERR_INVALID, "atp_get_unique_id: NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(ATP_ERR_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  std::memcpy(uid_out, &id, 128);
  return ATP_OK;
}

atp_status atp_mesh_init(int d1, int d2, int world_rank, const uint8_t uid[128], int cuda_device, atp_mesh** out) {
  if (uid == nullptr) return fail(ATP_ERR_INVALID, "atp_mesh_init: uid is NULL");
  return static_cast<atp_status>(atp::mesh_create(d1, d2, world_rank, uid, cuda_device, false, out));
}

atp_status atp_mesh_init_local(int d1, int d2, int rank, int cuda_device, atp_mesh** out) {
  return static_cast<atp_status>(atp::mesh_create(d1, d2, rank, nullptr, cuda_device, false, out));
}

atp_status atp_mesh_init_from_comms(int d1, int d2, int world_rank, void* dim1_comm, void* dim2_comm,
                                    int cuda_device, atp_mesh** out) {
  if ((d1 > 1 && dim1_comm == nullptr) || (d2 > 1 && dim2_comm == nullptr))
    return fail(ATP_ERR_INVALID, "atp_mesh_init_from_comms: a communicator of a dimension of size > 1 is NULL");
  atp_status s = static_cast<atp_status>(atp::mesh_create(d1, d2, world_rank, nullptr, cuda_device, false, out));
  if (s) return s;
  atp_mesh* m = *out;
  auto check_comm = [&](void* c, int size, int pos) {
    if (c == nullptr) return true;
    int cnt = 0, rk = -1;
    return ncclCommCount(static_cast<ncclComm_t>(c), &cnt) == ncclSuccess &&
           ncclCommUserRank(static_cast<ncclComm_t>(c), &rk) == ncclSuccess && cnt == size && rk == pos;
  };
  if (!check_comm(dim1_comm, d1, m->i1) || !check_comm(dim2_comm, d2, m->i2)) {
    atp::mesh_destroy(m);
    *out = nullptr;
    return fail(ATP_ERR_INVALID,
                "atp_mesh_init_from_comms: dim-1 comm must have d1 ranks with this rank at i1, dim-2 comm d2 ranks at i2");
  }
  m->dim1 = static_cast<ncclComm_t>(dim1_comm);
  m->dim2 = static_cast<ncclComm_t>(dim2_comm);
  m->comms_borrowed = true;
  m->local_only = false;
  m->comm_enabled = true;
  return ATP_OK;
}

atp_status atp_vmesh_init(int d1, int d2, int cuda_device, atp_mesh** out) {
  return static_cast<atp_status>(atp::mesh_create(d1, d2, 0, nullptr, cuda_device, true, out));
}

atp_status atp_mesh_destroy(atp_mesh* mesh) { return static_cast<atp_status>(atp::mesh_destroy(mesh)); }

atp_status atp_mesh_coords(const atp_mesh* mesh, int* i1, int* i2) {
  if (mesh == nullptr || i1 == nullptr || i2 == nullptr) return fail(ATP_ERR_INVALID, "atp_mesh_coords: NULL");
  if (mesh->is_virtual) return fail(ATP_ERR_INVALID, "atp_mesh_coords: virtual mesh has no single rank");
  *i1 = mesh->i1;
  *i2 = mesh->i2;
  return ATP_OK;
}

atp_status atp_mesh_dims(const atp_mesh* mesh, int* d1, int* d2, int* is_virtual) {
  if (mesh == nullptr) return fail(ATP_ERR_INVALID, "atp_mesh_dims: NULL");
  if (d1) *d1 = mesh->d1;
  if (d2) *d2 = mesh->d2;
  if (is_virtual) *is_virtual = mesh->is_virtual ? 1 : 0;
  return ATP_OK;
}

atp_status atp_mesh_groups(int d1, int d2, int dim, int* out) {
  if (d1 < 1 || d2 < 1 || out == nullptr) return fail(ATP_ERR_INVALID, "atp_mesh_groups: bad arguments");
  if (dim == 1) {
    int o = 0;
    for (int i2 = 0; i2 < d2; ++i2)
      for (int i1 = 0; i1 < d1; ++i1) out[o++] = i1 * d2 + i2;
    return ATP_OK;
  }
  if (dim == 2) {
    int o = 0;
    for (int i1 = 0; i1 < d1; ++i1)
      for (int i2 = 0; i2 < d2; ++i2) out[o++] = i1 * d2 + i2;
    return ATP_OK;
  }
  return fail(ATP_ERR_INVALID, "atp_mesh_groups: dim must be 1 or 2");
}

atp_status atp_mesh_enable_fused_ar(atp_mesh* mesh, size_t part_bytes) {
  if (mesh == nullptr || part_bytes == 0) return fail(ATP_ERR_INVALID, "atp_mesh_enable_fused_ar: bad arguments");
  if (mesh->capture_stream != nullptr) return fail(ATP_ERR_UNSUPPORTED, "atp_mesh_enable_fused_ar: mesh is capturing a graph");
  cudaSetDevice(mesh->device);
  return static_cast<atp_status>(atp::enable_fused_ar(mesh, part_bytes));
}

// Debug (not in atp.h's documented surface for users): device counters and host
// totals of one rank, copied on a separate stream (works while kernels spin).
extern "C" atp_status atp_debug_counters(atp_mesh* mesh, int rank, uint32_t* out, int n) {
  if (mesh == nullptr || out == nullptr || n < 1 || n > atp::kSigSlots) return fail(ATP_ERR_INVALID, "debug");
  return static_cast<atp_status>(atp::debug_counters(mesh, rank, out, n));
}

atp_status atp_mesh_set_gemm_ctas(atp_mesh* mesh, int max_ctas) {
  if (mesh == nullptr || max_ctas < 0) return fail(ATP_ERR_INVALID, "atp_mesh_set_gemm_ctas: bad arguments");
  mesh->gemm_ctas = max_ctas;
  return ATP_OK;
}

atp_status atp_mesh_set_gating(atp_mesh* mesh, int enabled) {
  if (mesh == nullptr) return fail(ATP_ERR_INVALID, "atp_mesh_set_gating: NULL mesh");
  mesh->gated = enabled != 0;
  return ATP_OK;
}

// ---------------------------------------------------------------- measurement hooks
atp_status atp_mesh_set_comm_enabled(atp_mesh* mesh, int enabled) {
  if (mesh == nullptr) return fail(ATP_ERR_INVALID, "atp_mesh_set_comm_enabled: NULL mesh");
  if (mesh->local_only && enabled) return fail(ATP_ERR_INVALID, "atp_mesh_set_comm_enabled: local mesh has no communicators");
  mesh->comm_enabled = enabled != 0;
  return ATP_OK;
}

atp_status atp_profile_begin(atp_mesh* mesh) {
  if (mesh == nullptr) return fail(ATP_ERR_INVALID, "atp_profile_begin: NULL mesh");
  if (mesh->capture_stream != nullptr) return fail(ATP_ERR_UNSUPPORTED, "atp_profile_begin: mesh is capturing a graph");
  mesh->profiling = true;
  mesh->prof_used = 0;
  return ATP_OK;
}

atp_status atp_profile_end(atp_mesh* mesh, atp_profile* out) {
  if (mesh == nullptr || out == nullptr) return fail(ATP_ERR_INVALID, "atp_profile_end: NULL argument");
  *out = atp_profile{};
  cudaSetDevice(mesh->device);
  for (size_t i = 0; i < mesh->prof_used; ++i) {
    const atp::ProfRec& r = mesh->prof[i];
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e != cudaSuccess) return fail(ATP_ERR_CUDA, std::string("atp_profile_end: ") + cudaGetErrorString(e));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    out->launches[r.cls] += 1;
    out->ms[r.cls] += ms;
    out->flops[r.cls] += r.flops;
    out->bytes[r.cls] += r.bytes;
  }
  mesh->profiling = false;
  mesh->prof_used = 0;
  return ATP_OK;
}

atp_status atp_profile_trace(atp_mesh* mesh, atp_trace_rec* out, int cap, int* n) {
  if (mesh == nullptr || n == nullptr || (cap > 0 && out == nullptr))
    return fail(ATP_ERR_INVALID, "atp_profile_trace: NULL argument");
  cudaSetDevice(mesh->device);
  *n = static_cast<int>(mesh->prof_used);
  for (size_t i = 0; i < mesh->prof_used && static_cast<int>(i) < cap; ++i) {
    const atp::ProfRec& r = mesh->prof[i];
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e != cudaSuccess) return fail(ATP_ERR_CUDA, std::string("atp_profile_trace: ") + cudaGetErrorString(e));
    float t0 = 0.f, t1 = 0.f;
    cudaEventElapsedTime(&t0, mesh->prof[0].a, r.a);
    cudaEventElapsedTime(&t1, mesh->prof[0].a, r.b);
    out[i] = atp_trace_rec{r.cls, r.stream, r.kind, r.sub, t0, t1};
  }
  return ATP_OK;
}

struct atp_graph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  uint64_t launches = 0;  // libatp kernels per replay (for atp_launch_count)
  int device = 0;
};

atp_status atp_graph_begin(atp_mesh* mesh, void* stream) {
  if (mesh == nullptr || stream == nullptr) return fail(ATP_ERR_INVALID, "atp_graph_begin: NULL mesh or stream");
  if (mesh->capture_stream != nullptr) return fail(ATP_ERR_INVALID, "atp_graph_begin: already capturing");
  if (mesh->profiling) return fail(ATP_ERR_UNSUPPORTED, "atp_graph_begin: mesh is profiling");
  for (const auto& r : mesh->rs)
    if (r.sym_base != nullptr)
      return fail(ATP_ERR_UNSUPPORTED, "atp_graph_begin: fused peer-memory all-reduce keeps cross-call state");
  cudaSetDevice(mesh->device);
  cudaError_t e = cudaStreamBeginCapture(static_cast<cudaStream_t>(stream), cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return fail(ATP_ERR_CUDA, std::string("cudaStreamBeginCapture: ") + cudaGetErrorString(e));
  mesh->capture_stream = stream;
  mesh->capture_launch0 = atp::launch_count();
  return ATP_OK;
}

atp_status atp_graph_end(atp_mesh* mesh, void* stream, atp_graph** out) {
  if (mesh == nullptr || out == nullptr || stream == nullptr || stream != mesh->capture_stream)
    return fail(ATP_ERR_INVALID, "atp_graph_end: not capturing on this stream");
  *out = nullptr;
  mesh->capture_stream = nullptr;
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(static_cast<cudaStream_t>(stream), &g);
  if (e != cudaSuccess || g == nullptr) {
    if (g) cudaGraphDestroy(g);
    return fail(ATP_ERR_CUDA, std::string("cudaStreamEndCapture: ") + cudaGetErrorString(e));
  }
  cudaGraphExec_t x = nullptr;
  e = cudaGraphInstantiate(&x, g, 0);
  if (e != cudaSuccess) {
    cudaGraphDestroy(g);
    return fail(ATP_ERR_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e));
  }
  auto* h = new atp_graph;
  h->graph = g;
  h->exec = x;
  h->launches = atp::launch_count() - mesh->capture_launch0;
  h->device = mesh->device;
  *out = h;
  return ATP_OK;
}

atp_status atp_graph_launch(atp_graph* graph, void* stream) {
  if (graph == nullptr) return fail(ATP_ERR_INVALID, "atp_graph_launch: NULL graph");
  cudaError_t e = cudaGraphLaunch(graph->exec, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(ATP_ERR_CUDA, std::string("cudaGraphLaunch: ") + cudaGetErrorString(e));
  atp::count_launch(graph->launches);
  return ATP_OK;
}

atp_status atp_graph_destroy(atp_graph* graph) {
  if (graph == nullptr) return ATP_OK;
  cudaSetDevice(graph->device);
  if (graph->exec) cudaGraphExecDestroy(graph->exec);
  if (graph->graph) cudaGraphDestroy(graph->graph);
  delete graph;
  return ATP_OK;
}

atp_status atp_launch_count(uint64_t* out) {
  if (out == nullptr) return fail(ATP_ERR_INVALID, "atp_launch_count: NULL");
  *out = atp::launch_count();
  return ATP_OK;
}

// ---------------------------------------------------------------- local GEMM
atp_status atp_gemm(const void* A, int64_t lda, int a_mn, const void* B, int64_t ldb, int b_mn, void* C, int64_t ldc,
                    int out_f32, const void* bias, int64_t M, int64_t N, int64_t K, int max_ctas, void* stream) {
  if (A == nullptr || B == nullptr || C == nullptr) return fail(ATP_ERR_INVALID, "atp_gemm: NULL operand");
  if (M <= 0 || N <= 0 || K <= 0 || M > (1 << 30) || N > (1 << 30) || K > (1 << 30))
    return fail(ATP_ERR_SHAPE, "atp_gemm: sizes out of range");
  if (ldc % 8 || !aligned16(C) || (bias && !aligned16(bias))) return fail(ATP_ERR_SHAPE, "atp_gemm: C/bias alignment");
  atp::GemmDesc d;
  d.max_ctas = max_ctas;
  d.epi = out_f32 ? atp::EPI_F32 : atp::EPI_BF16;
  d.ep.C = C;
  d.ep.ldc = ldc;
  d.ep.bias = bias;
  const char* m = atp::gemm_prepare(d, A, lda, a_mn != 0, B, ldb, b_mn != 0, (int)M, (int)N, (int)K);
  if (m) return fail(ATP_ERR_SHAPE, m);
  atp::count_launch(1);
  cudaError_t e = atp::gemm_launch(d, as_stream(stream));
  if (e != cudaSuccess) return fail(ATP_ERR_CUDA, std::string("atp_gemm: ") + cudaGetErrorString(e));
  return ATP_OK;
}

// ---------------------------------------------------------------- attention core
atp_status atp_attn_core_fwd(const void* qkv, int64_t ld_qkv, int64_t T, int64_t seq, int heads, int head_dim,
                             int causal, void* ctx, int64_t ld_ctx, float* lse, void* stream) {
  if (qkv == nullptr || ctx == nullptr || lse == nullptr) return fail(ATP_ERR_INVALID, "atp_attn_core_fwd: NULL buffer");
  if (const char* m = atp::attn_check(T, seq, heads, head_dim, ld_qkv, ld_ctx)) return fail(ATP_ERR_SHAPE, m);
  if (!aligned16(qkv) || !aligned16(ctx) || !aligned16(lse)) return fail(ATP_ERR_SHAPE, "atp_attn_core_fwd: alignment");
  atp::count_launch(1);
  cudaError_t e = atp::attn_fwd_launch(qkv, ld_qkv, static_cast<int>(T), static_cast<int>(seq), heads, causal, ctx,
                                       ld_ctx, lse, as_stream(stream));
  if (e != cudaSuccess) return fail(ATP_ERR_CUDA, std::string("atp_attn_core_fwd: ") + cudaGetErrorString(e));
  return ATP_OK;
}

size_t atp_attn_core_workspace(int64_t T, int heads) { return atp::attn_workspace_bytes(T, heads); }

atp_status atp_attn_core_bwd(const void* qkv, int64_t ld_qkv, const void* ctx, int64_t ld_ctx, const float* lse,
                             const void* dctx, int64_t ld_dctx, int64_t T, int64_t seq, int heads, int head_dim,
                             int causal, void* dqkv, int64_t ld_dqkv, void* workspace, size_t workspace_bytes,
                             void* stream) {
  if (!qkv || !ctx || !lse || !dctx || !dqkv || !workspace) return fail(ATP_ERR_INVALID, "atp_attn_core_bwd: NULL buffer");
  if (const char* m = atp::attn_check(T, seq, heads, head_dim, ld_qkv, ld_ctx)) return fail(ATP_ERR_SHAPE, m);
  if (ld_dctx < heads * 128 || ld_dctx % 8 || ld_dqkv < 3 * heads * 128 || ld_dqkv % 8)
    return fail(ATP_ERR_SHAPE, "atp_attn_core_bwd: dctx / dqkv pitch");
  if (workspace_bytes < atp::attn_workspace_bytes(T, heads)) return fail(ATP_ERR_SHAPE, "atp_attn_core_bwd: workspace too small");
  if (!aligned16(qkv) || !aligned16(ctx) || !aligned16(dctx) || !aligned16(dqkv) || !aligned16(workspace))
    return fail(ATP_ERR_SHAPE, "atp_attn_core_bwd: alignment");
  atp::count_launch(3);
  cudaError_t e = atp::attn_bwd_launch(qkv, ld_qkv, ctx, ld_ctx, lse, dctx, ld_dctx, static_cast<int>(T),
                                       static_cast<int>(seq), heads, causal, dqkv, ld_dqkv, workspace, as_stream(stream));
  if (e != cudaSuccess) return fail(ATP_ERR_CUDA, std::string("atp_attn_core_bwd: ") + cudaGetErrorString(e));
  return ATP_OK;
}

// ---------------------------------------------------------------- linears
static atp_status linear_fwd(atp_mesh* mesh, const atp_linear_fwd_args* args, int64_t M, int64_t K, int64_t N,
                             int chunks, atp_dtype dtype, void* stream, bool colfirst) {
  atp_status s = check_mesh(mesh, args);
  if (s) return s;
  if (dtype != ATP_BF16 && dtype != ATP_FP32) return fail(ATP_ERR_UNSUPPORTED, "linear: dtype must be ATP_BF16 or ATP_FP32");
  const int din = colfirst ? mesh->d2 : mesh->d1, dout = colfirst ? mesh->d1 : mesh->d2;
  if (chunks < 1 || chunks > atp::kMaxChunks || M < 1 || M % chunks || K % din || N % dout || !w8(K / din) ||
      !w8(N / dout))
    return fail(ATP_ERR_SHAPE,
                "linear fwd: need 1 <= chunks <= 16, M % chunks == 0, K % d_in == 0, N % d_out == 0, widths % 8 == 0");
  for (int r = 0; r < n_ranks(mesh); ++r)
    if (!args[r].x || !args[r].w || !args[r].y) return fail(ATP_ERR_INVALID, "linear fwd: NULL buffer");
  return run(mesh, stream, [&](const atp::RankView& rv, int r, Sched& out) {
    return atp::build_linear_fwd(rv, colfirst, args[r], M, K, N, chunks, dtype, out);
  });
}

static atp_status linear_bwd(atp_mesh* mesh, const atp_linear_bwd_args* args, int64_t M, int64_t K, int64_t N,
                             int chunks, atp_dtype dtype, void* stream, bool colfirst) {
  atp_status s = check_mesh(mesh, args);
  if (s) return s;
  if (dtype != ATP_BF16 && dtype != ATP_FP32) return fail(ATP_ERR_UNSUPPORTED, "linear: dtype must be ATP_BF16 or ATP_FP32");
  const int din = colfirst ? mesh->d2 : mesh->d1, dout = colfirst ? mesh->d1 : mesh->d2;
  if (chunks < 1 || chunks > atp::kMaxChunks || M < 1 || M % chunks || K % din || N % dout || !w8(K / din) ||
      !w8(N / dout) || M % 8)
    return fail(ATP_ERR_SHAPE,
                "linear bwd: need 1 <= chunks <= 16, M % chunks == 0, M % 8 == 0, K % d_in, N % d_out, widths % 8 == 0");
  for (int r = 0; r < n_ranks(mesh); ++r)
    if (!args[r].x || !args[r].w || !args[r].dy || !args[r].dx) return fail(ATP_ERR_INVALID, "linear bwd: NULL buffer");
  return run(mesh, stream, [&](const atp::RankView& rv, int r, Sched& out) {
    return atp::build_linear_bwd(rv, colfirst, args[r], M, K, N, chunks, dtype, out);
  });
}

atp_status atp_linear_colfirst_fwd(atp_mesh* mesh, const atp_linear_fwd_args* args, int64_t M, int64_t K, int64_t N,
                                   int chunks, atp_dtype dtype, void* stream) {
  return linear_fwd(mesh, args, M, K, N, chunks, dtype, stream, true);
}
atp_status atp_linear_rowfirst_fwd(atp_mesh* mesh, const atp_linear_fwd_args* args, int64_t M, int64_t K, int64_t N,
                                   int chunks, atp_dtype dtype, void* stream) {
  return linear_fwd(mesh, args, M, K, N, chunks, dtype, stream, false);
}
atp_status atp_linear_colfirst_bwd(atp_mesh* mesh, const atp_linear_bwd_args* args, int64_t M, int64_t K, int64_t N,
                                   int chunks, atp_dtype dtype, void* stream) {
  return linear_bwd(mesh, args, M, K, N, chunks, dtype, stream, true);
}
atp_status atp_linear_rowfirst_bwd(atp_mesh* mesh, const atp_linear_bwd_args* args, int64_t M, int64_t K, int64_t N,
                                   int chunks, atp_dtype dtype, void* stream) {
  return linear_bwd(mesh, args, M, K, N, chunks, dtype, stream, false);
}

// ---------------------------------------------------------------- composites
static atp_status check_layer_shapes(const atp_mesh* m, int64_t T, int64_t h, int64_t F, int64_t heads, int chunks,
                                     bool attn, bool mlp) {
  if (chunks < 1 || chunks > atp::kMaxChunks || T < 1 || h < 1 || T % chunks || (T / chunks) % 8 || h % m->d2 ||
      !w8(h / m->d2))
    return fail(ATP_ERR_SHAPE,
                "layer: need 1 <= chunks <= 16, T % chunks == 0, (T/chunks) % 8 == 0, h % d2 == 0, (h/d2) % 8 == 0");
  if (mlp && (F < 1 || F % m->d1 || !w8(F / m->d1)))
    return fail(ATP_ERR_SHAPE, "mlp: need F % d1 == 0 and (F/d1) % 8 == 0");
  if (attn && (heads < 1 || heads % m->d1 || h % heads || (h / heads) % 8 || !w8(h / m->d1)))
    return fail(ATP_ERR_SHAPE, "attn: need heads % d1 == 0, h % heads == 0, head dim % 8 == 0, (h/d1) % 8 == 0");
  return ATP_OK;
}

atp_status atp_mlp_fwd(atp_mesh* mesh, const atp_mlp_fwd_args* args, int64_t T, int64_t h, int64_t F, int chunks,
                       atp_dtype dtype, void* stream) {
  atp_status s = check_mesh(mesh, args);
  if (s) return s;
  if (dtype != ATP_BF16 && dtype != ATP_FP32) return fail(ATP_ERR_UNSUPPORTED, "mlp: dtype must be ATP_BF16 or ATP_FP32");
  if ((s = check_layer_shapes(mesh, T, h, F, 1, chunks, false, true))) return s;
  for (int r = 0; r < n_ranks(mesh); ++r) {
    const auto& a = args[r];
    if (!a.x || !a.w1 || !a.w2 || !a.u || !a.h_act || !a.z) return fail(ATP_ERR_INVALID, "mlp fwd: NULL buffer");
  }
  return run(mesh, stream, [&](const atp::RankView& rv, int r, Sched& out) {
    atp::LayerParts p;
    p.mlp_fwd = &args[r];
    return atp::build_layer(rv, p, T, h, F, 1, chunks, dtype, out);
  });
}

atp_status atp_mlp_bwd(atp_mesh* mesh, const atp_mlp_bwd_args* args, int64_t T, int64_t h, int64_t F, int chunks,
                       atp_dtype dtype, void* stream) {
  atp_status s = check_mesh(mesh, args);
  if (s) return s;
  if (dtype != ATP_BF16 && dtype != ATP_FP32) return fail(ATP_ERR_UNSUPPORTED, "mlp: dtype must be ATP_BF16 or ATP_FP32");
  if ((s = check_layer_shapes(mesh, T, h, F, 1, chunks, false, true))) return s;
  for (int r = 0; r < n_ranks(mesh); ++r) {
    const auto& a = args[r];
    if (!a.x || !a.w1 || !a.w2 || !a.u || !a.h_act || !a.dz || !a.dx || !a.ws_dh)
      return fail(ATP_ERR_INVALID, "mlp bwd: NULL buffer");
  }
  return run(mesh, stream, [&](const atp::RankView& rv, int r, Sched& out) {
    atp::LayerParts p;
    p.mlp_bwd = &args[r];
    return atp::build_layer(rv, p, T, h, F, 1, chunks, dtype, out);
  });
}

atp_status atp_attn_proj_fwd(atp_mesh* mesh, const atp_attn_fwd_args* args, int64_t T, int64_t h, int64_t heads,
                             int chunks, atp_core core, atp_dtype dtype, void* stream) {
  atp_status s = check_mesh(mesh, args);
  if (s) return s;
  if (dtype != ATP_BF16 && dtype != ATP_FP32) return fail(ATP_ERR_UNSUPPORTED, "attn: dtype must be ATP_BF16 or ATP_FP32");
  if (core != ATP_CORE_SUM_QKV) return fail(ATP_ERR_UNSUPPORTED, "attn: only ATP_CORE_SUM_QKV");
  if ((s = check_layer_shapes(mesh, T, h, 8, heads, chunks, true, false))) return s;
  for (int r = 0; r < n_ranks(mesh); ++r) {
    const auto& a = args[r];
    if (!a.x || !a.wqkv || !a.wo || !a.qkv || !a.ctx || !a.y) return fail(ATP_ERR_INVALID, "attn fwd: NULL buffer");
  }
  return run(mesh, stream, [&](const atp::RankView& rv, int r, Sched& out) {
    atp::LayerParts p;
    p.attn_fwd = &args[r];
    return atp::build_layer(rv, p, T, h, 8, heads, chunks, dtype, out);
  });
}

atp_status atp_attn_proj_bwd(atp_mesh* mesh, const atp_attn_bwd_args* args, int64_t T, int64_t h, int64_t heads,
                             int chunks, atp_core core, atp_dtype dtype, void* stream) {
  atp_status s = check_mesh(mesh, args);
  if (s) return s;
  if (dtype != ATP_BF16 && dtype != ATP_FP32) return fail(ATP_ERR_UNSUPPORTED, "attn: dtype must be ATP_BF16 or ATP_FP32");
  if (core != ATP_CORE_SUM_QKV) return fail(ATP_ERR_UNSUPPORTED, "attn: only ATP_CORE_SUM_QKV");
  if ((s = check_layer_shapes(mesh, T, h, 8, heads, chunks, true, false))) return s;
  for (int r = 0; r < n_ranks(mesh); ++r) {
    const auto& a = args[r];
    if (!a.x || !a.wqkv || !a.wo || !a.ctx || !a.dy || !a.dx || !a.ws_dctx || !a.ws_dqkv)
      return fail(ATP_ERR_INVALID, "attn bwd: NULL buffer");
  }
  return run(mesh, stream, [&](const atp::RankView& rv, int r, Sched& out) {
    atp::LayerParts p;
    p.attn_bwd = &args[r];
    return atp::build_layer(rv, p, T, h, 8, heads, chunks, dtype, out);
  });
}

atp_status atp_layer_fwd_bwd(atp_mesh* mesh, const atp_layer_args* args, int64_t T, int64_t h, int64_t F,
                             int64_t heads, int chunks, int do_backward, atp_dtype dtype, void* stream) {
  atp_status s = check_mesh(mesh, args);
  if (s) return s;
  if (dtype != ATP_BF16 && dtype != ATP_FP32) return fail(ATP_ERR_UNSUPPORTED, "layer: dtype must be ATP_BF16 or ATP_FP32");
  if ((s = check_layer_shapes(mesh, T, h, F, heads, chunks, true, true))) return s;
  for (int r = 0; r < n_ranks(mesh); ++r) {
    const auto& a = args[r];
    if (a.mlp.x != a.attn.y) return fail(ATP_ERR_INVALID, "layer: mlp.x must equal attn.y");
    if (do_backward && (a.attn_b.dy != a.mlp_b.dx || a.mlp_b.x != a.attn.y))
      return fail(ATP_ERR_INVALID, "layer: attn_b.dy must equal mlp_b.dx and mlp_b.x must equal attn.y");
  }
  return run(mesh, stream, [&](const atp::RankView& rv, int r, Sched& out) {
    atp::LayerParts p;
    p.attn_fwd = &args[r].attn;
    p.mlp_fwd = &args[r].mlp;
    if (do_backward) {
      p.mlp_bwd = &args[r].mlp_b;
      p.attn_bwd = &args[r].attn_b;
    }
    return atp::build_layer(rv, p, T, h, F, heads, chunks, dtype, out);
  });
}

atp_status atp_layer_stack_fwd_bwd(atp_mesh* mesh, const atp_layer_args* args, int n_layers, int64_t T, int64_t h,
                                   int64_t F, int64_t heads, int chunks, atp_dtype dtype, void* stream) {
  atp_status s = check_mesh(mesh, args);
  if (s) return s;
  if (n_layers < 1) return fail(ATP_ERR_INVALID, "layer stack: n_layers must be >= 1");
  if (dtype != ATP_BF16 && dtype != ATP_FP32) return fail(ATP_ERR_UNSUPPORTED, "layer stack: dtype must be ATP_BF16 or ATP_FP32");
  if ((s = check_layer_shapes(mesh, T, h, F, heads, chunks, true, true))) return s;
  const int n = n_ranks(mesh);
  for (int l = 0; l < n_layers; ++l)
    for (int r = 0; r < n; ++r) {
      const auto& a = args[l * n + r];
      if (a.mlp.x != a.attn.y || a.attn_b.dy != a.mlp_b.dx || a.mlp_b.x != a.attn.y)
        return fail(ATP_ERR_INVALID, "layer stack: each layer must chain as in atp_layer_fwd_bwd");
      if (l + 1 < n_layers) {
        const auto& nx = args[(l + 1) * n + r];
        if (nx.attn.x != a.mlp.z || a.mlp_b.dz != nx.attn_b.dx)
          return fail(ATP_ERR_INVALID, "layer stack: layer l+1 attn.x must be layer l mlp.z and layer l mlp_b.dz "
                                       "must be layer l+1 attn_b.dx");
      }
    }
  return run(mesh, stream, [&](const atp::RankView& rv, int r, Sched& out) {
    std::vector<atp::LayerParts> parts(n_layers);
    for (int l = 0; l < n_layers; ++l) {
      const auto& a = args[l * n + r];
      parts[l].attn_fwd = &a.attn;
      parts[l].mlp_fwd = &a.mlp;
      parts[l].mlp_bwd = &a.mlp_b;
      parts[l].attn_bwd = &a.attn_b;
    }
    return atp::build_layer_stack(rv, parts.data(), n_layers, T, h, F, heads, chunks, dtype, out);
  });
}

// ---------------------------------------------------------------- workspace sizes
atp_status atp_workspace_size(int op, int d1, int d2, int64_t T, int64_t h, int64_t F, int64_t heads, int64_t seq,
                              int chunks, size_t bytes[4]) {
  if (bytes == nullptr || d1 < 1 || d2 < 1 || T < 1 || h < 1 || F < 1) return fail(ATP_ERR_INVALID, "atp_workspace_size: bad arguments");
  bytes[0] = bytes[1] = bytes[2] = bytes[3] = 0;
  const size_t t = static_cast<size_t>(T);
  const size_t dh = t * (F / d1) * 2, dctx = t * (h / d1) * 2, dqkv = t * (3 * h / d1) * 2;
  switch (op) {
    case ATP_OP_MLP_BWD: bytes[0] = dh; break;
    case ATP_OP_ATTN_BWD: bytes[0] = dctx; bytes[1] = dqkv; break;
    case ATP_OP_LAYER: bytes[0] = dh; bytes[1] = dctx; bytes[2] = dqkv; break;
    case ATP_OP_GPT_LAYER:
      if (heads < 1 || seq < 1 || chunks < 1) return fail(ATP_ERR_INVALID, "atp_workspace_size: heads, seq, chunks");
      bytes[0] = atp::gpt_workspace_bytes(d1, d2, T, h, F, heads, seq, chunks);
      break;
    default: return fail(ATP_ERR_INVALID, "atp_workspace_size: unknown op");
  }
  return ATP_OK;
}

// ---------------------------------------------------------------- full GPT layer
size_t atp_gpt_workspace(int d1, int d2, int64_t T, int64_t h, int64_t F, int64_t heads, int64_t seq, int chunks) {
  if (d1 < 1 || d2 < 1 || chunks < 1 || T < 1) return 0;
  return atp::gpt_workspace_bytes(d1, d2, T, h, F, heads, seq, chunks);
}

atp_status atp_gpt_layer_fwd_bwd(atp_mesh* mesh, const atp_gpt_args* args, int64_t T, int64_t h, int64_t F,
                                 int64_t heads, int64_t seq, int chunks, int causal, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  atp_status s = check_mesh(mesh, args);
  if (s) return s;
  const int d1 = mesh->d1, d2 = mesh->d2;
  if (heads < 1 || h % heads || h / heads != 128) return fail(ATP_ERR_SHAPE, "gpt layer: head dim h/heads must be 128");
  if (heads % (d1 * d2)) return fail(ATP_ERR_SHAPE, "gpt layer: heads % (d1*d2) != 0 (heads are sharded over both dims)");
  if (h % d2 || (3 * h) % d1 || F % d1 || (F / d1) % 8 || (h / d2) % 8)
    return fail(ATP_ERR_SHAPE, "gpt layer: h % d2, F % d1 and 8-element local widths required");
  if (seq < 128 || seq % 128) return fail(ATP_ERR_SHAPE, "gpt layer: seq must be a multiple of 128");
  if (chunks < 1 || chunks > atp::kMaxChunks || T % (static_cast<int64_t>(chunks) * seq))
    return fail(ATP_ERR_SHAPE, "gpt layer: T % (chunks * seq) != 0 (chunks are whole sequences) or chunks > 16");
  const size_t per = atp::gpt_workspace_bytes(d1, d2, T, h, F, heads, seq, chunks);
  const int n = n_ranks(mesh);
  if (workspace == nullptr || workspace_bytes < per * n) return fail(ATP_ERR_SHAPE, "gpt layer: workspace too small");
  for (int r = 0; r < n; ++r) {
    const atp_gpt_args& a = args[r];
    const void* req[] = {a.x, a.dz, a.g1, a.be1, a.g2, a.be2, a.wqkv, a.bqkv, a.wo, a.bo, a.w1, a.b1, a.w2, a.b2,
                         a.a, a.sv1, a.qkv, a.lse, a.ctx, a.y1, a.bn, a.sv2, a.u, a.h, a.z, a.dx,
                         a.dwqkv, a.dbqkv, a.dwo, a.dbo, a.dw1, a.db1, a.dw2, a.db2, a.dg1, a.dbe1, a.dg2, a.dbe2};
    for (const void* p : req)
      if (p == nullptr) return fail(ATP_ERR_INVALID, "gpt layer: NULL buffer");
    if (d2 > 1 && a.ctx_loc == nullptr) return fail(ATP_ERR_INVALID, "gpt layer: ctx_loc required when d2 > 1");
  }
  char* ws = static_cast<char*>(workspace);
  return run(mesh, stream, [&](const atp::RankView& rv, int r, Sched& out) {
    return atp::build_gpt_layer(rv, args[r], T, h, F, heads, seq, chunks, causal, ws + per * r, out);
  });
}

// ---------------------------------------------------------------- probe
atp_status atp_probe_allreduce(atp_mesh* mesh, int dim, size_t msg_bytes, int iters, void* buf, double* busbw_gbps,
                               double* algbw_gbps, double* seconds) {
  if (mesh == nullptr || buf == nullptr || iters < 1 || msg_bytes < 2 || (dim != 1 && dim != 2))
    return fail(ATP_ERR_INVALID, "atp_probe_allreduce: bad arguments");
  if (mesh->is_virtual || mesh->local_only) return fail(ATP_ERR_INVALID, "atp_probe_allreduce: needs a distributed mesh");
  const int p = dim == 1 ? mesh->d1 : mesh->d2;
  if (busbw_gbps) *busbw_gbps = 0.0;
  if (algbw_gbps) *algbw_gbps = 0.0;
  if (seconds) *seconds = 0.0;
  if (p == 1) return ATP_OK;
  cudaSetDevice(mesh->device);
  ncclComm_t comm = dim == 1 ? mesh->dim1 : mesh->dim2;
  cudaStream_t st = mesh->rs[0].comm;
  const size_t count = msg_bytes / 2;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  ncclResult_t r = ncclAllReduce(buf, buf, count, ncclBfloat16, ncclSum, comm, st);  // warm-up
  cudaEventRecord(a, st);
  for (int i = 0; i < iters && r == ncclSuccess; ++i) r = ncclAllReduce(buf, buf, count, ncclBfloat16, ncclSum, comm, st);
  cudaEventRecord(b, st);
  cudaError_t e = cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (r != ncclSuccess) return fail(ATP_ERR_NCCL, std::string("probe: ") + ncclGetErrorString(r));
  if (e != cudaSuccess) return fail(ATP_ERR_CUDA, std::string("probe: ") + cudaGetErrorString(e));
  const double t = (ms * 1e-3) / iters;
  const double alg = static_cast<double>(count * 2) / t / 1e9;
  if (algbw_gbps) *algbw_gbps = alg;
  if (busbw_gbps) *busbw_gbps = alg * 2.0 * (p - 1) / p;
  if (seconds) *seconds = t;
  return ATP_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- HCM probe
namespace {

// Time `iters` in-place all-reduces of `bytes` on `comm` (every rank of the
// parent communicator calls this together); returns seconds per all-reduce.
double time_allreduce(ncclComm_t comm, void* buf, size_t bytes, int iters, cudaStream_t st, ncclResult_t* err) {
  const size_t count = bytes / 2;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  *err = ncclAllReduce(buf, buf, count, ncclBfloat16, ncclSum, comm, st);  // warm-up
  cudaEventRecord(a, st);
  for (int i = 0; i < iters && *err == ncclSuccess; ++i) *err = ncclAllReduce(buf, buf, count, ncclBfloat16, ncclSum, comm, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return (ms * 1e-3) / iters;
}

}  // namespace

extern "C" atp_status atp_probe_hcm(atp_mesh* world, const size_t* msg_bytes, int n_msgs, size_t calib_bytes,
                                    int iters, void* scratch, atp_hcm* hcm_out, double* p2p_matrix,
                                    atp_calib* calib_out) {
  if (world == nullptr || world->is_virtual || world->local_only || msg_bytes == nullptr || n_msgs < 1 ||
      iters < 1 || scratch == nullptr || hcm_out == nullptr || calib_bytes < 2)
    return fail(ATP_ERR_INVALID, "atp_probe_hcm: needs a distributed mesh, message sizes, scratch and outputs");
  cudaSetDevice(world->device);
  const int N = world->d1 * world->d2;
  const int me = world->rank;
  cudaStream_t st = world->rs[0].comm;
  ncclResult_t r = ncclSuccess;
  auto nccl_fail = [&](const char* what) { return fail(ATP_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r)); };
  auto busbw = [&](ncclComm_t c, int p, size_t bytes) {
    const double t = time_allreduce(c, scratch, bytes, iters, st, &r);
    return p > 1 ? (static_cast<double>(bytes) / t) * 2.0 * (p - 1) / p / 1e9 : 0.0;
  };
  // group bandwidth: N-rank all-reduce on the world communicator; every rank
  // takes the slowest rank's figure (min over ranks, exchanged as an exact
  // double) so all ranks hold the same HCM and search alike
  double group = 0.0;
  for (int i = 0; i < n_msgs && N > 1; ++i) {
    const double b = busbw(world->world, N, msg_bytes[i]);
    if (r != ncclSuccess) return nccl_fail("probe group");
    group = b > group ? b : group;
  }
  if (N > 1) {
    double v = -group;  // max of -bw = min of bw
    double* d = static_cast<double*>(scratch);
    cudaMemcpyAsync(d, &v, sizeof(v), cudaMemcpyHostToDevice, st);
    r = ncclAllReduce(d, d, 1, ncclFloat64, ncclMax, world->world, st);
    if (r != ncclSuccess) return nccl_fail("probe group exchange");
    cudaMemcpyAsync(&v, d, sizeof(v), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    group = -v;
  }
  // P2P: round-robin tournament (circle method) over N (or N+1 with a bye) slots
  const int slots = N + (N & 1);
  std::vector<double> pm(static_cast<size_t>(N) * N, 0.0);
  for (int round = 0; round < slots - 1 && N > 1; ++round) {
    // slot -> rank: slot 0 fixed, others rotate
    auto rank_at = [&](int slot) { return slot == 0 ? 0 : 1 + ((slot - 1 + round) % (slots - 1)); };
    int partner = -1, color = -1;
    for (int k = 0; k < slots / 2; ++k) {
      const int a = rank_at(k), b = rank_at(slots - 1 - k);
      if (a == me && b < N) partner = b, color = k;
      if (b == me && a < N) partner = a, color = k;
    }
    ncclComm_t pc = nullptr;
    r = ncclCommSplit(world->world, partner >= 0 ? color : NCCL_SPLIT_NOCOLOR, me, &pc, nullptr);
    if (r != ncclSuccess) return nccl_fail("probe pair split");
    if (pc != nullptr) {
      double best = 0.0;
      for (int i = 0; i < n_msgs; ++i) {
        const double b = busbw(pc, 2, msg_bytes[i]);
        if (r != ncclSuccess) return nccl_fail("probe pair");
        best = b > best ? b : best;
      }
      pm[static_cast<size_t>(me) * N + partner] = best;
      ncclCommDestroy(pc);
    }
  }
  // every rank learns the full matrix: all-reduce the (disjoint) rows in fp32 via NCCL
  {
    std::vector<float> h(static_cast<size_t>(N) * N);
    for (size_t i = 0; i < h.size(); ++i) h[i] = static_cast<float>(pm[i]);
    float* d = static_cast<float*>(scratch);
    cudaMemcpyAsync(d, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice, st);
    r = ncclAllReduce(d, d, h.size(), ncclFloat32, ncclSum, world->world, st);
    if (r != ncclSuccess) return nccl_fail("probe matrix exchange");
    cudaMemcpyAsync(h.data(), d, h.size() * sizeof(float), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    for (size_t i = 0; i < h.size(); ++i) pm[i] = h[i];
  }
  double p2p_min = 0.0;
  bool have = false;
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j)
      if (i != j) {
        const double v = 0.5 * (pm[static_cast<size_t>(i) * N + j] + pm[static_cast<size_t>(j) * N + i]);
        if (!have || v < p2p_min) p2p_min = v;
        have = true;
      }
  if (p2p_matrix != nullptr)
    for (size_t i = 0; i < pm.size(); ++i) p2p_matrix[i] = pm[i];
  *hcm_out = atp_hcm{};
  hcm_out->n_layers = 1;
  hcm_out->ranks[0] = N;
  hcm_out->p2p_gbps[0] = N > 1 ? p2p_min : 1.0;
  hcm_out->group_gbps[0] = N > 1 ? group : 1.0;
  // calibration: every mesh of N, both dimensions, all groups concurrently
  if (calib_out != nullptr) {
    *calib_out = atp_calib{};
    for (int d1 = N; d1 >= 1 && calib_out->n < ATP_MAX_PLAN; --d1) {
      if (N % d1) continue;
      const int d2 = N / d1;
      const int i1 = me / d2, i2 = me % d2;
      double bk[2] = {0.0, 0.0};
      for (int dim = 1; dim <= 2; ++dim) {
        const int p = dim == 1 ? d1 : d2;
        ncclComm_t c = nullptr;
        r = ncclCommSplit(world->world, dim == 1 ? i2 : i1, dim == 1 ? i1 : i2, &c, nullptr);
        if (r != ncclSuccess) return nccl_fail("probe calibration split");
        if (p > 1) {
          const double t = time_allreduce(c, scratch, calib_bytes, iters, st, &r);
          if (r != ncclSuccess) return nccl_fail("probe calibration");
          bk[dim - 1] = static_cast<double>(calib_bytes) / t / 1e9;
        }
        ncclCommDestroy(c);
      }
      // every rank reports the slowest group: take the max time = min bandwidth over ranks
      float v[2] = {static_cast<float>(bk[0] > 0 ? 1.0 / bk[0] : 0.0), static_cast<float>(bk[1] > 0 ? 1.0 / bk[1] : 0.0)};
      float* d = static_cast<float*>(scratch);
      cudaMemcpyAsync(d, v, sizeof(v), cudaMemcpyHostToDevice, st);
      r = ncclAllReduce(d, d, 2, ncclFloat32, ncclMax, world->world, st);
      if (r != ncclSuccess) return nccl_fail("probe calibration exchange");
      cudaMemcpyAsync(v, d, sizeof(v), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      const int k = calib_out->n++;
      calib_out->d1[k] = d1;
      calib_out->d2[k] = d2;
      calib_out->b1[k] = v[0] > 0 ? 1.0 / v[0] : 0.0;
      calib_out->b2[k] = v[1] > 0 ? 1.0 / v[1] : 0.0;
    }
  }
  return ATP_OK;
}
