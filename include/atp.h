/*
 * atp.h — C ABI of libatp: the B200-native hot path of ATP, Adaptive Tensor
 * Parallelism (arXiv 2301.08658).  "P:n" cites /root/reference/PAPER.md line n.
 *
 * The library implements the column-first / row-first tensor-parallel
 * transformer linear block on a DeviceMesh(d1, d2), forward and backward,
 * with chunk-based communication/computation overlap, plus the paper's
 * communication cost model and mesh search.
 *
 * Conventions (all entry points)
 *   - Status codes, never exceptions or aborts.  On failure atp_last_error()
 *     returns a thread-local message.  Shapes are validated BEFORE anything is
 *     enqueued, so a failed call has no device side effects.
 *   - Device pointers: bf16 (`ATP_BF16`) row-major, contiguous rows, 16-byte
 *     aligned.  The caller owns every buffer (activations, weights, saved
 *     tensors, gradients, workspace) and the stream; the library owns only the
 *     communicators it creates, its communication stream(s) and its events.
 *   - Calls are asynchronous: they enqueue on the caller's `stream` and return;
 *     results are valid in stream order.  No hidden allocation on the hot path.
 *   - Weights are in math orientation W[in, out] (y = x W), sharded per P:218:
 *       column-first W: [Shard(1), Shard(0)] -> local [in/d2, out/d1]
 *       row-first    W: [Shard(0), Shard(1)] -> local [in/d1, out/d2]
 *     Activations between blocks are [Replicate, Shard(1)]: rank
 *     (i1, i2) holds the column block i2, i.e. a local [T, h/d2] matrix.
 *   - rank = i1*d2 + i2.  Dim-1 groups = ranks sharing i2 (d1 members);
 *     dim-2 groups = ranks sharing i1 (d2 members).
 *   - Mesh handles come in two kinds.  A *distributed* mesh (atp_mesh_init)
 *     is one rank of an SPMD job, one process per GPU, collectives through
 *     NCCL; the per-rank argument pointer `args` points to ONE struct.  A
 *     *virtual* mesh (atp_vmesh_init) holds all d1*d2 ranks in one process on
 *     one device (test/validation vehicle: same schedule, same kernels, the
 *     group sums done by a library kernel); `args` points to an ARRAY of d1*d2
 *     structs in rank order.
 */
#ifndef ATP_H_
#define ATP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ATP_VERSION "0.1.0"

typedef enum {
  ATP_OK = 0,
  ATP_ERR_INVALID = 1,     /* bad argument (mesh size, dim, null pointer ...) */
  ATP_ERR_SHAPE = 2,       /* divisibility / alignment precondition violated  */
  ATP_ERR_CUDA = 3,        /* CUDA runtime error                              */
  ATP_ERR_NCCL = 4,        /* NCCL error                                      */
  ATP_ERR_EMPTY = 5,       /* search: no admissible candidate mesh            */
  ATP_ERR_UNSUPPORTED = 6  /* feature not built / not available              */
} atp_status;

/* ATP_BF16: the product path (bf16 storage, tcgen05 GEMMs, fp32 accumulation,
 * bf16 all-reduce).  ATP_FP32: check mode — every activation, weight, bias and
 * workspace buffer is fp32, GEMMs are CUDA-core fp32 FMA, all-reduces fp32;
 * same schedule, so the sharded pipeline can be checked against the fp64
 * oracle at <= 1e-4 (north_star). */
typedef enum { ATP_BF16 = 0, ATP_FP32 = 1 } atp_dtype;

typedef struct atp_mesh atp_mesh; /* opaque */

const char* atp_last_error(void);
const char* atp_version(void);

/* ------------------------------------------------------------------ mesh
 * DeviceMesh(d1, d2).  atp_get_unique_id fills 128 bytes (an
 * ncclUniqueId) on rank 0; the caller broadcasts them (e.g. over
 * torch.distributed) and every rank calls atp_mesh_init with the same bytes.
 * The library creates the world communicator on `cuda_device`, splits it into
 * the dim-1 communicator (color = i2, key = i1) and the dim-2 communicator
 * (color = i1, key = i2), and creates its communication stream and events.
 * Errors: ATP_ERR_INVALID if d1 < 1, d2 < 1 or world_rank out of range;
 * ATP_ERR_NCCL / ATP_ERR_CUDA on library failures.
 */
atp_status atp_get_unique_id(uint8_t uid_out[128]);
atp_status atp_mesh_init(int d1, int d2, int world_rank, const uint8_t uid[128], int cuda_device,
                         atp_mesh** out);
/* All d1*d2 ranks of a mesh in this process on `cuda_device` (see header). */
/* Borrow the caller's communicators (SURVEY §8(b) variant): dim1_comm holds
 * the d1 ranks sharing this rank's i2 (this rank at position i1), dim2_comm
 * the d2 ranks sharing i1 (at position i2), with rank = i1*d2 + i2;
 * ncclComm_t values passed as void*.  A comm of a size-1 dimension may be
 * NULL.  The mesh never destroys borrowed comms; features that need a world
 * communicator (atp_mesh_enable_fused_ar on a multi-rank mesh, probes) return
 * an error.  Errors: ATP_ERR_INVALID (NULL comm of a dimension > 1, comm size
 * or rank position not matching). */
atp_status atp_mesh_init_from_comms(int d1, int d2, int world_rank, void* dim1_comm, void* dim2_comm,
                                    int cuda_device, atp_mesh** out);
atp_status atp_vmesh_init(int d1, int d2, int cuda_device, atp_mesh** out);
/* Dry-run handle for ONE rank `rank` of DeviceMesh(d1, d2) on `cuda_device`
 * without communicators: every all-reduce of its schedule is elided (results
 * are therefore not the mesh's results).  Used to measure, on one GPU, the
 * compute part of a rank's step for a mesh that needs d1*d2 GPUs. */
atp_status atp_mesh_init_local(int d1, int d2, int rank, int cuda_device, atp_mesh** out);
atp_status atp_mesh_destroy(atp_mesh* mesh);
/* Coordinates of a distributed mesh's rank (virtual mesh: ATP_ERR_INVALID). */
atp_status atp_mesh_coords(const atp_mesh* mesh, int* i1, int* i2);
atp_status atp_mesh_dims(const atp_mesh* mesh, int* d1, int* d2, int* is_virtual);
/* Pure: groups of mesh dimension `dim` (1 or 2), written as consecutive
 * member lists into out[d1*d2] (dim 1: d2 groups of d1; dim 2: d1 groups of
 * d2), members in ascending mesh coordinate. */
atp_status atp_mesh_groups(int d1, int d2, int dim, int* out);
/* Cap the CTAs of the persistent GEMMs (0 = all SMs) so that an overlapped
 * NCCL kernel keeps SMs of its own (SURVEY §7 "SM sharing"). */
atp_status atp_mesh_set_gemm_ctas(atp_mesh* mesh, int max_ctas);

/* Chunk-gated GEMMs (opt-in; initial value from env ATP_GATED=1).  When on,
 * and the GEMM CTA cap leaves at least 16 SMs free, a stage that follows a
 * signalled stage launches ONE GEMM whose producer waits per chunk for the
 * previous stage's chunk gate (written after that chunk's all-reduce and
 * elementwise step) instead of the stream waiting for its last all-reduce.
 * Same results.  Errors: ATP_ERR_INVALID (NULL mesh). */
atp_status atp_mesh_set_gating(atp_mesh* mesh, int enabled);

/* Fused GEMM -> all-reduce -> elementwise stages over peer memory (opt-in;
 * PAPER.md §4.1 P:337 names GEMM/all-reduce fusion as the alternative to
 * chunking — here the two compose).  Allocates this rank's peer-visible
 * buffer (two receive regions of `part_bytes` each — one stage's [T, width]
 * bf16, laid out as p sender slots of T/p rows — plus counters) and maps the
 * buffers of its dim-1 and dim-2 group members (CUDA IPC handles all-gathered
 * over the world communicator; a virtual mesh uses the other virtual ranks'
 * buffers).  Collective on a distributed mesh.  Afterwards every
 * communicating bf16 stage whose chunk splits into p slices of whole 128-row
 * tiles (p <= 8) runs as: the GEMM stores each output tile with TMA straight
 * into the receive slot of the member owning the tile's row slice (the
 * reduce-scatter's data movement, tile by tile, over NVLink) and counts it on
 * that member's chunk counter; then per chunk ONE kernel per member sums its
 * slice of the p partials, applies the post-all-reduce elementwise step, and
 * pulls the other members' reduced slices with bulk copies (all-gather) —
 * 2(p-1)/p of the chunk per member, no NCCL call on the data path.  Stages
 * that do not qualify use the NCCL path.  Errors: ATP_ERR_INVALID (already
 * enabled, or a mesh dimension above 16), ATP_ERR_CUDA, ATP_ERR_NCCL. */
atp_status atp_mesh_enable_fused_ar(atp_mesh* mesh, size_t part_bytes);

/* Measurement hooks (bench.py).  atp_mesh_set_comm_enabled(mesh, 0) replaces
 * every all-reduce by a no-op (events still recorded, so the schedule and its
 * dependencies are unchanged): the comm-disabled twin of SURVEY §8(d) that
 * gives exposed communication = t(layer) - t(layer, comm disabled); results
 * are then wrong by construction.  atp_profile_begin(mesh) makes the executor
 * bracket every kernel / all-reduce it enqueues with CUDA timing events on the
 * stream it is launched on; atp_profile_end synchronises on those events and
 * returns, per class (0 = tcgen05 GEMM, 1 = elementwise / LayerNorm,
 * 2 = collective, 3 = attention core), the launch count, summed device
 * milliseconds, and the algorithmic FLOPs (GEMM: 2MNK; attention: 4 d per
 * visible (query, key) pair forward, 2.5x that backward) and bytes (GEMM:
 * A+B+C; elementwise: reads+writes; all-reduce: ring bytes sent
 * 2(p-1)/p*n*esz; reduce-scatter / all-gather: (p-1)*block*esz) of those
 * launches.  atp_launch_count() is a
 * process-wide count of kernels libatp has launched (NCCL's not included). */
typedef struct {
  int64_t launches[4];
  double ms[4];
  double flops[4];
  double bytes[4];
} atp_profile;

atp_status atp_mesh_set_comm_enabled(atp_mesh* mesh, int enabled);
/* Diagnostics: copies rank `rank`'s first n chunk counters (device) into
 * out[0..n) and the host-side targets into out[n..2n), on a separate stream,
 * so it works while a schedule is stuck waiting on a counter. */
atp_status atp_debug_counters(atp_mesh* mesh, int rank, uint32_t* out, int n);
atp_status atp_profile_begin(atp_mesh* mesh);
atp_status atp_profile_end(atp_mesh* mesh, atp_profile* out);
/* Per-op timeline of the profiled region (call before atp_profile_end, which
 * resets it): for each bracketed launch in enqueue order, its class (as
 * above), stream (0 compute, 1 communication, 2 auxiliary), op kind (GEMM,
 * elementwise, collective, fused all-reduce), sub-kind (GEMM epilogue /
 * elementwise kind / collective kind) and start / end in device milliseconds
 * from the first record's start.  Writes min(cap, records) entries to out and
 * the record count to *n.  Synchronises on the events. */
typedef struct {
  int cls, stream, kind, sub;
  double t0_ms, t1_ms;
} atp_trace_rec;
atp_status atp_profile_trace(atp_mesh* mesh, atp_trace_rec* out, int cap, int* n);
atp_status atp_launch_count(uint64_t* out);

/* ------------------------------------------------------------------ CUDA graphs
 * Capture a sequence of calls on one mesh (e.g. one atp_layer_fwd_bwd, or a
 * stack of layers) into a CUDA graph and replay it: one cudaGraphLaunch per
 * step instead of the host building and enqueuing every GEMM, elementwise
 * step, stream wait and collective (NCCL calls are captured as graph nodes).
 *   atp_graph_begin(mesh, stream): starts stream capture (thread-local mode) on
 *     `stream`; the calls that follow enqueue into the capture.  Make one
 *     uncaptured call with the same arguments first (first-use setup).
 *   atp_graph_end(mesh, stream, &g): ends the capture, instantiates the graph.
 *   atp_graph_launch(g, stream): replays it (asynchronous, stream order).  The
 *     captured calls read and write the same device buffers on every replay.
 *   atp_graph_destroy(g).
 * Every call starts from zeroed chunk counters (no state carried between
 * calls), so replays are independent.  Not available while profiling, or on a
 * mesh with the fused peer-memory all-reduce (its counters are shared with
 * peers): ATP_ERR_UNSUPPORTED.  Errors: ATP_ERR_INVALID, ATP_ERR_CUDA (capture
 * or instantiation failed; the capture is ended and discarded). */
typedef struct atp_graph atp_graph;
atp_status atp_graph_begin(atp_mesh* mesh, void* stream);
atp_status atp_graph_end(atp_mesh* mesh, void* stream, atp_graph** out);
atp_status atp_graph_launch(atp_graph* graph, void* stream);
atp_status atp_graph_destroy(atp_graph* graph);

/* ------------------------------------------------------------------ local GEMM
 * One local shard contraction on the tcgen05 tensor cores (the building block
 * of F3/F6/F8/F11 and of dX = dY W^T, dW = X^T dY):
 *     C[M,N] = A[M,K] * B[N,K]^T (+ bias[N]),  bf16 in, fp32 accumulate.
 * a_mn = 0: A stored row-major [M,K] with pitch lda; 1: A stored [K,M].
 * b_mn = 0: B stored row-major [N,K] with pitch ldb; 1: B stored [K,N].
 * out_f32 = 1 writes fp32 C (pitch ldc), else bf16.  (a_mn, b_mn) = (1, 0)
 * is unsupported.  N, K multiples of 8 (M too when a_mn); A, B, C, bias 16-byte
 * aligned and ldc a multiple of 8 (C is written with TMA bulk tensor stores);
 * else ATP_ERR_SHAPE.  max_ctas = 0: all SMs.
 */
atp_status atp_gemm(const void* A, int64_t lda, int a_mn, const void* B, int64_t ldb, int b_mn,
                    void* C, int64_t ldc, int out_f32, const void* bias, int64_t M, int64_t N,
                    int64_t K, int max_ctas, void* stream);

/* ------------------------------------------------------------------ attention core
 * Softmax attention of one rank's heads (Eq. 1):
 * for every sequence n (rows [n*seq, (n+1)*seq) of the T token rows) and head j,
 *     O = softmax(Q K^T / sqrt(d)) V        (causal: key t' > query t masked)
 * on tcgen05 tensor cores.  qkv [T, 3*heads*d] bf16, row pitch ld_qkv, columns
 * head-interleaved (head j: q at 3jd, k at 3jd+d, v at 3jd+2d; reading G19).
 * ctx [T, heads*d] bf16 (pitch ld_ctx) receives O; lse [heads][T] fp32 receives
 * the natural-log log-sum-exp of each row's scaled, masked scores (saved for
 * the backward).  Caller-owned device buffers; asynchronous on `stream`.
 * Requirements: head_dim == 128, seq % 128 == 0, T % seq == 0, pitches
 * multiples of 8 elements, 16-byte aligned pointers; else ATP_ERR_SHAPE.
 */
atp_status atp_attn_core_fwd(const void* qkv, int64_t ld_qkv, int64_t T, int64_t seq, int heads, int head_dim,
                             int causal, void* ctx, int64_t ld_ctx, float* lse, void* stream);

/* Backward of atp_attn_core_fwd (dV = P^T dO, dP = dO V^T, dS = P*(dP - D),
 * D = rowsum(dO*O), dQ = dS K/sqrt(d), dK = dS^T Q/sqrt(d)): dqkv [T,
 * 3*heads*d] bf16 (pitch ld_dqkv, same column order as qkv) from the forward's
 * qkv, ctx (= O) and lse and the upstream dctx [T, heads*d] (pitch ld_dctx).
 * `workspace` (device, caller-owned) must hold atp_attn_core_workspace(T,
 * heads) bytes (fp32 dQ accumulator and D); its contents are scratch.
 * Same shape requirements as the forward; ATP_ERR_SHAPE otherwise. */
atp_status atp_attn_core_bwd(const void* qkv, int64_t ld_qkv, const void* ctx, int64_t ld_ctx, const float* lse,
                             const void* dctx, int64_t ld_dctx, int64_t T, int64_t seq, int heads, int head_dim,
                             int causal, void* dqkv, int64_t ld_dqkv, void* workspace, size_t workspace_bytes,
                             void* stream);
size_t atp_attn_core_workspace(int64_t T, int heads);

/* ------------------------------------------------------------------ linears
 * Column-first TP linear (Fig. 5 right): x [M, K/d2] ([Replicate,
 * Shard(1)]), w [K/d2, N/d1] ([Shard(1), Shard(0)]), bias [N/d1] or NULL;
 * y [M, N/d1] = all-reduce over mesh dim 2 of x w (+ bias once), i.e.
 * [Shard(1), Replicate].  Row-first (Fig. 5 left): x [M, K/d1]
 * ([Shard(1), Replicate]), w [K/d1, N/d2], y [M, N/d2] all-reduced over dim 1
 * ([Replicate, Shard(1)]).  The M rows are processed in `chunks` chunks; the
 * all-reduce of chunk k overlaps the GEMM of chunk k+1 (§4.1).
 * Backward: dx = all-reduce over the conjugate dim (column-first: 1,
 * row-first: 2) of dy w^T; dw = x^T dy (fp32, local, no communication);
 * dbias = column sums of dy (fp32) or NULL.  The dw GEMM runs after the dx
 * chunks are enqueued so it overlaps their all-reduces (§4.2).
 * Errors: ATP_ERR_SHAPE if K % d, N % d, M % chunks, or the 8-element
 * alignment of the GEMM fails.
 */
typedef struct {
  const void* x;
  const void* w;
  const void* bias; /* may be NULL */
  void* y;
} atp_linear_fwd_args;

typedef struct {
  const void* x;  /* saved forward input */
  const void* w;
  const void* dy;
  void* dx;       /* bf16 */
  float* dw;      /* fp32 */
  float* dbias;   /* fp32 or NULL */
} atp_linear_bwd_args;

atp_status atp_linear_colfirst_fwd(atp_mesh* mesh, const atp_linear_fwd_args* args, int64_t M,
                                   int64_t K, int64_t N, int chunks, atp_dtype dtype, void* stream);
atp_status atp_linear_rowfirst_fwd(atp_mesh* mesh, const atp_linear_fwd_args* args, int64_t M,
                                   int64_t K, int64_t N, int chunks, atp_dtype dtype, void* stream);
atp_status atp_linear_colfirst_bwd(atp_mesh* mesh, const atp_linear_bwd_args* args, int64_t M,
                                   int64_t K, int64_t N, int chunks, atp_dtype dtype, void* stream);
atp_status atp_linear_rowfirst_bwd(atp_mesh* mesh, const atp_linear_bwd_args* args, int64_t M,
                                   int64_t K, int64_t N, int chunks, atp_dtype dtype, void* stream);

/* ------------------------------------------------------------------ composites
 * Feed-forward block (Fig. 6b): FC1 column-first + f3 (dim 2),
 * U = . + b1 (saved), H = GeLU(U) (exact erf, saved), FC2 row-first + f4
 * (dim 1), Z = X + . + b2 (residual added after the all-reduce).
 * Local shapes (T tokens, h, F): x, z, dz, dx [T, h/d2]; w1 [h/d2, F/d1];
 * b1 [F/d1]; w2 [F/d1, h/d2]; b2 [h/d2]; u, h_act [T, F/d1];
 * dw1 fp32 [h/d2, F/d1]; db1 fp32 [F/d1]; dw2 fp32 [F/d1, h/d2]; db2 fp32 [h/d2];
 * workspace dh [T, F/d1] bf16.
 * Errors: ATP_ERR_SHAPE unless h % d2 == 0, F % d1 == 0, T % chunks == 0 and
 * all local widths are multiples of 8.
 */
typedef struct {
  const void* x; const void* w1; const void* b1; const void* w2; const void* b2;
  void* u; void* h_act; void* z;
} atp_mlp_fwd_args;

typedef struct {
  const void* x; const void* w1; const void* w2; const void* u; const void* h_act; const void* dz;
  void* dx; float* dw1; float* db1; float* dw2; float* db2;
  void* ws_dh;
} atp_mlp_bwd_args;

atp_status atp_mlp_fwd(atp_mesh* mesh, const atp_mlp_fwd_args* args, int64_t T, int64_t h,
                       int64_t F, int chunks, atp_dtype dtype, void* stream);
atp_status atp_mlp_bwd(atp_mesh* mesh, const atp_mlp_bwd_args* args, int64_t T, int64_t h,
                       int64_t F, int chunks, atp_dtype dtype, void* stream);

/* Attention projections (Fig. 6a): QKV column-first + f1 (dim 2), the
 * attention core, Output row-first + f2 (dim 1), Y = X + . + bo.
 * Wqkv columns are head-interleaved (head*3d + {q,k,v}*d + j) so that the
 * column-first split gives rank i1 the heads [i1*a/d1, (i1+1)*a/d1).
 * core = ATP_CORE_SUM_QKV: zero-FLOP stand-in ctx = Q + K + V per head
 * (the softmax core of Eq. 1 is outside this path).
 * Local shapes: x, y, dy, dx [T, h/d2]; wqkv [h/d2, 3h/d1]; bqkv [3h/d1];
 * wo [h/d1, h/d2]; bo [h/d2]; qkv [T, 3h/d1]; ctx [T, h/d1];
 * dwqkv fp32 [h/d2, 3h/d1]; dbqkv fp32 [3h/d1]; dwo fp32 [h/d1, h/d2];
 * dbo fp32 [h/d2]; workspaces dctx [T, h/d1], dqkv [T, 3h/d1] bf16.
 * Errors: ATP_ERR_SHAPE unless heads % d1 == 0, h % heads == 0, h % d2 == 0,
 * T % chunks == 0 and local widths are multiples of 8.
 */
typedef enum { ATP_CORE_SUM_QKV = 0 } atp_core;

typedef struct {
  const void* x; const void* wqkv; const void* bqkv; const void* wo; const void* bo;
  void* qkv; void* ctx; void* y;
} atp_attn_fwd_args;

typedef struct {
  const void* x; const void* wqkv; const void* wo; const void* ctx; const void* dy;
  void* dx; float* dwqkv; float* dbqkv; float* dwo; float* dbo;
  void* ws_dctx; void* ws_dqkv;
} atp_attn_bwd_args;

atp_status atp_attn_proj_fwd(atp_mesh* mesh, const atp_attn_fwd_args* args, int64_t T, int64_t h,
                             int64_t heads, int chunks, atp_core core, atp_dtype dtype,
                             void* stream);
atp_status atp_attn_proj_bwd(atp_mesh* mesh, const atp_attn_bwd_args* args, int64_t T, int64_t h,
                             int64_t heads, int chunks, atp_core core, atp_dtype dtype,
                             void* stream);

/* Whole linear block of one GPT layer, forward then backward, as ONE chunk
 * pipeline: chunk k of a block waits only on chunk k's all-reduce of the
 * block before it (Fig. 7; reading G14), so the last all-reduce of the
 * attention block overlaps the first FC1 GEMM.  Shapes as above (F = ffn). */
typedef struct {
  atp_attn_fwd_args attn;   /* attn.y is the MLP input (y1)              */
  atp_mlp_fwd_args mlp;     /* mlp.x must equal attn.y                   */
  atp_mlp_bwd_args mlp_b;   /* mlp_b.dz = upstream grad, mlp_b.dx = dy1  */
  atp_attn_bwd_args attn_b; /* attn_b.dy must equal mlp_b.dx             */
} atp_layer_args;

atp_status atp_layer_fwd_bwd(atp_mesh* mesh, const atp_layer_args* args, int64_t T, int64_t h,
                             int64_t F, int64_t heads, int chunks, int do_backward,
                             atp_dtype dtype, void* stream);

/* A stack of n_layers identical-shape layers, forward 0..n-1 then backward
 * n-1..0, as ONE chunk pipeline (SURVEY §8(d) L_bench; Fig. 7): layer
 * l+1's first GEMM waits only on layer l's last stage, so a layer's last
 * all-reduce overlaps the next layer's first GEMM instead of draining at a
 * call boundary.  args = [n_layers][local ranks] (layer-major).  Chaining
 * (checked, ATP_ERR_INVALID otherwise): layer l+1's attn.x is layer l's
 * mlp.z, and layer l's mlp_b.dz is layer l+1's attn_b.dx (the gradient of
 * its input); each layer also satisfies atp_layer_fwd_bwd's rules.  Same
 * shapes / errors as atp_layer_fwd_bwd; backward always runs. */
atp_status atp_layer_stack_fwd_bwd(atp_mesh* mesh, const atp_layer_args* args, int n_layers, int64_t T,
                                   int64_t h, int64_t F, int64_t heads, int chunks, atp_dtype dtype,
                                   void* stream);

/* ------------------------------------------------------------------ workspace sizes
 * Bytes of every caller-allocated workspace buffer of an op, in the order the
 * op's argument struct names them (the library makes no hidden allocations):
 *   ATP_OP_MLP_BWD   [ws_dh]                       (T x F/d1 bf16)
 *   ATP_OP_ATTN_BWD  [ws_dctx, ws_dqkv]            (T x h/d1, T x 3h/d1 bf16)
 *   ATP_OP_LAYER     [ws_dh, ws_dctx, ws_dqkv]
 *   ATP_OP_GPT_LAYER [workspace of atp_gpt_layer_fwd_bwd, per rank]
 * Unused entries are 0.  heads/seq/chunks matter only for ATP_OP_GPT_LAYER.
 * Pure host computation.  Errors: ATP_ERR_INVALID. */
typedef enum { ATP_OP_MLP_BWD = 0, ATP_OP_ATTN_BWD = 1, ATP_OP_LAYER = 2, ATP_OP_GPT_LAYER = 3 } atp_op;
atp_status atp_workspace_size(int op, int d1, int d2, int64_t T, int64_t h, int64_t F, int64_t heads, int64_t seq,
                              int chunks, size_t bytes[4]);

/* ------------------------------------------------------------------ full GPT layer
 * One pre-LN GPT layer, forward then backward, on DeviceMesh(d1, d2) (SURVEY
 * §8(f) NEXT #1; readings G29-G35 in DESIGN.md):
 *   A = LN1(X); QKV = A Wqkv + bqkv; ctx = softmax-attention(QKV) (Eq. 1,
 *   P:83, causal); Y1 = X + ctx Wo + bo; B = LN2(Y1); U = B W1 + b1;
 *   H = GeLU(U); Z = Y1 + H W2 + b2; then the backward for upstream dZ.
 * The attention core is fully sharded (Fig. 6(a)): the QKV partial
 * sums are reduce-scattered over mesh dim 2 so rank (i1, i2) holds heads
 * [(i1*d2 + i2)*hl, +hl), hl = heads/(d1*d2); ctx is all-gathered over dim 2
 * before Out; backward reduce-scatters dctx and all-gathers dQKV on dim 2.
 * LayerNorm statistics are all-reduced over dim 2 ([rows, 2] fp32).  Chunks
 * are whole sequences: T = b*seq, T % (chunks*seq) == 0 (reading G34).
 * Local shapes (hc = h/d2, h1 = h/d1, q1 = 3h/d1, F1 = F/d1, ql = q1/d2,
 * cl = h1/d2), bf16 unless noted:
 *   inputs   x, dz [T, hc]; g1, be1, g2, be2 [hc]; wqkv [hc, q1]; bqkv [q1];
 *            wo [h1, hc]; bo [hc]; w1 [hc, F1]; b1 [F1]; w2 [F1, hc]; b2 [hc]
 *   saved    a, y1, bn [T, hc]; sv1, sv2 fp32 [T, 2] (mean, rstd);
 *            qkv [T, ql]; ctx_loc [T, cl]; lse fp32 [T*hl]; ctx [T, h1];
 *            u, h [T, F1]
 *   outputs  z, dx [T, hc]; fp32 grads dwqkv [hc, q1], dbqkv [q1],
 *            dwo [h1, hc], dbo [hc], dw1 [hc, F1], db1 [F1], dw2 [F1, hc],
 *            db2 [hc], dg1, dbe1, dg2, dbe2 [hc]
 *   workspace  atp_gpt_workspace(...) bytes (device, caller-owned scratch).
 * With d2 == 1, ctx_loc may equal ctx.  bf16 only.  Requirements: head dim
 * h/heads == 128, heads % (d1*d2) == 0, seq % 128 == 0, T % (chunks*seq) ==
 * 0, h % d2 == 0, widths multiples of 8; else ATP_ERR_SHAPE. */
typedef struct {
  const void* x; const void* dz;
  const void* g1; const void* be1; const void* g2; const void* be2;
  const void* wqkv; const void* bqkv; const void* wo; const void* bo;
  const void* w1; const void* b1; const void* w2; const void* b2;
  void* a; float* sv1; void* qkv; void* ctx_loc; float* lse; void* ctx;
  void* y1; void* bn; float* sv2; void* u; void* h;
  void* z; void* dx;
  float* dwqkv; float* dbqkv; float* dwo; float* dbo; float* dw1; float* db1; float* dw2; float* db2;
  float* dg1; float* dbe1; float* dg2; float* dbe2;
} atp_gpt_args;

size_t atp_gpt_workspace(int d1, int d2, int64_t T, int64_t h, int64_t F, int64_t heads, int64_t seq, int chunks);
atp_status atp_gpt_layer_fwd_bwd(atp_mesh* mesh, const atp_gpt_args* args, int64_t T, int64_t h, int64_t F,
                                 int64_t heads, int64_t seq, int chunks, int causal, void* workspace,
                                 size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------ cost model
 * Hierarchical communication matrix (§3.4): layers outermost
 * first; layer j: R_j ranks, P2P bandwidth between two layer-j ranks and the
 * group bandwidth of one layer-j rank, GB/s per direction.
 */
#define ATP_MAX_HCM_LAYERS 8
#define ATP_MAX_PLAN 64

typedef struct {
  int n_layers;
  int ranks[ATP_MAX_HCM_LAYERS];
  double p2p_gbps[ATP_MAX_HCM_LAYERS];
  double group_gbps[ATP_MAX_HCM_LAYERS];
} atp_hcm;

typedef struct {
  int64_t L, b, s, h, heads, bytes_per_elem;
} atp_model;

/* Measured algorithm bandwidths (P:482 calibration, reading G11); a value
 * <= 0 means "not calibrated" for that dimension. */
typedef struct {
  int n;
  int d1[ATP_MAX_PLAN], d2[ATP_MAX_PLAN];
  double b1[ATP_MAX_PLAN], b2[ATP_MAX_PLAN];
} atp_calib;

typedef struct {
  int d1, d2;
  double b1_prime, b2_prime; /* Eq. 3 (GB/s); 0 when NoComm or calibrated */
  double b1, b2;             /* Eq. 4 algorithm bandwidth (GB/s); 0 = NoComm */
  double t_f[4];             /* Eq. 2 terms f1..f4 (seconds, x 2Lbs*bytes)   */
  double t_comm;             /* seconds                                      */
  int calibrated;
} atp_cost;

typedef struct {
  int n_ranked;
  atp_cost ranked[ATP_MAX_PLAN]; /* ascending t_comm; ties: larger d1 first */
  int chosen;                    /* index into ranked (always 0)            */
  int n_rejected;
  int rejected_d1[ATP_MAX_PLAN], rejected_d2[ATP_MAX_PLAN];
} atp_plan;

/* ATP mesh search (§3.5): Eq. 3 -> Eq. 4 -> Eq. 2 for every
 * (d1, d2) with d1*d2 = n_devices (= product of HCM ranks), argmin T_comm.
 * calib may be NULL.  Deterministic; doubles evaluated in the canonical order
 * documented in DESIGN.md so they equal the oracle's bit for bit.
 * Errors: ATP_ERR_INVALID (HCM product != n_devices, non-positive bandwidth,
 * bad model); ATP_ERR_EMPTY if no mesh is admissible. */
atp_status atp_search(const atp_hcm* hcm, const atp_model* model, int n_devices,
                      const atp_calib* calib, atp_plan* out);

/* Eq. 3 alone for one mesh (NoComm -> 0). ATP_ERR_SHAPE on misalignment. */
atp_status atp_effective_bandwidth(const atp_hcm* hcm, int d1, int d2, double* b1_prime,
                                   double* b2_prime);

/* Executed collective list of one layer fwd+bwd (reading G4): up to `cap`
 * entries of (phase 0=fwd/1=bwd, block 0=qkv/1=out/2=fc1/3=fc2, dim, p,
 * elements per rank); *n_calls = the full count.  Totals are int64 exact. */
typedef struct {
  int phase, block, dim, p;
  int64_t elems;
} atp_call;

atp_status atp_comm_volume(int d1, int d2, int64_t T, int64_t h, int64_t F, int chunks,
                           atp_call* calls, int cap, int* n_calls, int64_t* dim1_elems,
                           int64_t* dim2_elems);

/* Chunk-overlap timing model (§4.1 Fig. 7, §4.2; SPEC's overlap
 * module): one compute and one communication stream; stage i has compute
 * comp[i] (its GEMM over all chunks), extra compute dw[i] after it on the
 * compute stream (§4.2's dW GEMM) and all-reduce time comm[i]; chunks split
 * comp and comm evenly.  mode 0 = signalled stages (the next stage's GEMM waits
 * for the last all-reduce of the previous stage), 1 = per-chunk (chunk k waits
 * for chunk k's all-reduce, Fig. 7).  Outputs the makespan and the exposed
 * communication (makespan - total compute), in the inputs' time unit.
 * Pure host code; bit-identical to oracle/overlap.py. */
atp_status atp_overlap_estimate(int n_stages, const double* comp, const double* dw, const double* comm, int chunks,
                                int mode, double* makespan, double* exposed);

/* Chunk-count planner (§4.1 P:332 fixes c by hand,
 * "2 or 4"; Table 3 P:449 shows the best c depends on the interconnect).
 * atp_layer_stages splits one layer fwd+bwd on DeviceMesh(d1, d2) into its 8
 * linear stages in schedule order (QKV, Out, FC1, FC2 forward; FC2, FC1, Out,
 * QKV backward): comp[i] = compute_ms x (stage GEMM FLOPs / all GEMM FLOPs),
 * dw[i] = compute_ms x (dW GEMM FLOPs / all; backward stages only, §4.2),
 * comm[i] = executed ring all-reduce bytes 2(p-1)/p x T x width x bytes_per_elem
 * (the atp_comm_volume list, reading G4) / busbw_gbps, in ms; 0 on a size-1
 * dimension.  Output arrays hold 8 doubles (caller-owned host memory).
 * atp_plan_chunks evaluates atp_overlap_estimate (mode 0 signalled / 1
 * per-chunk) on those stages for each candidate chunk count chunks[i]
 * (ascending, dividing T) with its measured compute-side time compute_ms[i]
 * (collectives elided), writes makespan_ms[i] / exposed_ms[i] (either may be
 * NULL) and *chosen = the count with the smallest makespan (ties -> fewer
 * chunks).  Pure host code, bit-identical to oracle/overlap.py layer_stages /
 * plan_chunks.  Errors: ATP_ERR_INVALID (shapes not divisible by the mesh,
 * busbw <= 0, bad candidates). */
atp_status atp_layer_stages(int d1, int d2, int64_t T, int64_t h, int64_t F, int bytes_per_elem, double compute_ms,
                            double busbw_gbps, double* comp, double* dw, double* comm);
atp_status atp_plan_chunks(int d1, int d2, int64_t T, int64_t h, int64_t F, int bytes_per_elem, int n_cand,
                           const int* chunks, const double* compute_ms, double busbw_gbps, int mode, int* chosen,
                           double* makespan_ms, double* exposed_ms);

/* ------------------------------------------------------------------ probe
 * Bandwidth probe feeding the HCM (§3.4) and the calibration, on a
 * distributed mesh spanning all ranks: times ncclAllReduce on each mesh
 * dimension's communicator with every group active concurrently.
 * msg_bytes: message size per rank; result bus bandwidths (GB/s, per
 * direction, = algBW * 2(p-1)/p) for dim 1 and dim 2 (0 if size 1), and the
 * algorithm bandwidths (bytes / time).  Collective call: all ranks. */
atp_status atp_probe_allreduce(atp_mesh* mesh, int dim, size_t msg_bytes, int iters, void* buf,
                               double* busbw_gbps, double* algbw_gbps, double* seconds);

/* Full probe (S1 of SURVEY §8(a)) on a distributed mesh spanning all N ranks
 * (any d1 x d2 = N; collective call on every rank):
 *   - group bandwidth: busBW of the N-rank all-reduce (GroupBW of the
 *     single-layer HCM of an NVSwitch node);
 *   - P2P: busBW of concurrent 2-rank all-reduces, all pairs covered by a
 *     round-robin schedule of N-1 rounds (pairs of one round run together);
 *     reported as the minimum over pairs (p2p_min) and the full matrix
 *     (p2p_matrix[N*N], GB/s, diagonal 0; may be NULL);
 *   - calibration: for every mesh (d1', d2') of N, all dim-1 groups
 *     then all dim-2 groups all-reduce `calib_bytes` per rank concurrently;
 *     B_k = algorithm bandwidth (bytes / time, GB/s), NoComm dims report 0.
 * Messages: bus bandwidth is the max over sizes in msg_bytes[0..n_msgs).
 * hcm_out receives ONE layer {N, p2p_min, group}.  `scratch` is a device
 * buffer of at least max(msg_bytes, calib_bytes) bytes.
 * Errors: ATP_ERR_INVALID (virtual/local mesh, bad sizes), ATP_ERR_NCCL. */
atp_status atp_probe_hcm(atp_mesh* world, const size_t* msg_bytes, int n_msgs, size_t calib_bytes, int iters,
                         void* scratch, atp_hcm* hcm_out, double* p2p_matrix, atp_calib* calib_out);

#ifdef __cplusplus
}
#endif
#endif /* ATP_H_ */
