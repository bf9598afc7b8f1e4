"""Thin Python binding over libatp (same names as include/atp.h).

Argument marshalling only: every step of the hot path runs in libatp's CUDA
kernels / NCCL calls.  PyTorch supplies device memory, streams and (in
bench.py) the process group used to broadcast the NCCL unique id.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

from . import _abi
from ._abi import AtpError, check, lib
from . import layout


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


# ------------------------------------------------------------------ mesh
def atp_get_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().atp_get_unique_id(buf))
    return buf.raw


class Mesh:
    """DeviceMesh(d1, d2) handle.  ``Mesh.virtual`` holds all ranks in this
    process on one GPU; ``Mesh.distributed`` is one rank of an SPMD job."""

    def __init__(self, handle, d1: int, d2: int, is_virtual: bool, rank: int = 0):
        self.handle = handle
        self.d1, self.d2 = d1, d2
        self.is_virtual = is_virtual
        self.rank = rank

    @classmethod
    def virtual(cls, d1: int, d2: int, device: int = 0) -> "Mesh":
        h = C.c_void_p()
        check(lib().atp_vmesh_init(d1, d2, device, C.byref(h)))
        return cls(h, d1, d2, True)

    @classmethod
    def local(cls, d1: int, d2: int, rank: int, device: int = 0) -> "Mesh":
        """Dry-run handle of one rank (collectives elided) for single-GPU measurement."""
        h = C.c_void_p()
        check(lib().atp_mesh_init_local(d1, d2, rank, device, C.byref(h)))
        return cls(h, d1, d2, False, rank)

    @classmethod
    def distributed(cls, d1: int, d2: int, rank: int, uid: bytes, device: int) -> "Mesh":
        h = C.c_void_p()
        check(lib().atp_mesh_init(d1, d2, rank, uid, device, C.byref(h)))
        return cls(h, d1, d2, False, rank)

    @classmethod
    def from_comms(cls, d1: int, d2: int, rank: int, dim1_comm: int, dim2_comm: int, device: int) -> "Mesh":
        """Mesh over the caller's NCCL communicators (ncclComm_t values as ints; borrowed, not destroyed)."""
        h = C.c_void_p()
        check(lib().atp_mesh_init_from_comms(d1, d2, rank, dim1_comm, dim2_comm, device, C.byref(h)))
        return cls(h, d1, d2, False, rank)

    @property
    def n_local_ranks(self) -> int:
        return self.d1 * self.d2 if self.is_virtual else 1

    def local_ranks(self) -> list[int]:
        return list(range(self.d1 * self.d2)) if self.is_virtual else [self.rank]

    def coords(self) -> tuple[int, int]:
        i1, i2 = C.c_int(), C.c_int()
        check(lib().atp_mesh_coords(self.handle, C.byref(i1), C.byref(i2)))
        return i1.value, i2.value

    def set_gemm_ctas(self, n: int) -> None:
        check(lib().atp_mesh_set_gemm_ctas(self.handle, n))

    def set_gating(self, on: bool) -> None:
        """Chunk-gated GEMMs (opt-in; needs a GEMM CTA cap leaving >= 16 SMs free)."""
        check(lib().atp_mesh_set_gating(self.handle, 1 if on else 0))

    def enable_fused_ar(self, part_bytes: int) -> None:
        """Opt in to the fused peer-memory all-reduce (collective on a distributed mesh)."""
        check(lib().atp_mesh_enable_fused_ar(self.handle, part_bytes))

    def destroy(self) -> None:
        if self.handle:
            check(lib().atp_mesh_destroy(self.handle))
            self.handle = None


def atp_mesh_groups(d1: int, d2: int, dim: int) -> list[list[int]]:
    out = (C.c_int * (d1 * d2))()
    check(lib().atp_mesh_groups(d1, d2, dim, out))
    flat = list(out)
    size = d1 if dim == 1 else d2
    return [flat[i:i + size] for i in range(0, len(flat), size)]


# ------------------------------------------------------------------ local GEMM
def atp_gemm(A, B, Cout, a_mn: bool = False, b_mn: bool = False, bias=None, max_ctas: int = 0, stream=None):
    """Cout[M,N] = A[M,K] B[N,K]^T (+bias) on the tcgen05 tensor cores.

    a_mn: A is given as its transpose [K,M]; b_mn: B given as [K,N]."""
    import torch

    M, N = Cout.shape
    K = A.shape[0] if a_mn else A.shape[1]
    check(lib().atp_gemm(A.data_ptr(), A.stride(0), int(a_mn), B.data_ptr(), B.stride(0), int(b_mn),
                         Cout.data_ptr(), Cout.stride(0), int(Cout.dtype == torch.float32), _ptr(bias),
                         M, N, K, max_ctas, _stream(stream)))


# ------------------------------------------------------------------ attention core
def atp_attn_core_fwd(qkv, ctx, lse, seq: int, heads: int, causal: bool = True, head_dim: int = 128, stream=None):
    """ctx[T, heads*d] = softmax(Q K^T / sqrt(d)) V per sequence/head of the
    head-interleaved qkv[T, 3*heads*d]; lse[heads, T] (fp32) = row log-sum-exp."""
    T = qkv.shape[0]
    check(lib().atp_attn_core_fwd(qkv.data_ptr(), qkv.stride(0), T, seq, heads, head_dim, int(causal),
                                  ctx.data_ptr(), ctx.stride(0), lse.data_ptr(), _stream(stream)))


def atp_attn_core_bwd(qkv, ctx, lse, dctx, dqkv, seq: int, heads: int, causal: bool = True, workspace=None,
                      head_dim: int = 128, stream=None):
    """dqkv = d(attention)/d(qkv) for upstream dctx (forward's qkv, ctx, lse)."""
    import torch

    T = qkv.shape[0]
    nbytes = lib().atp_attn_core_workspace(T, heads)
    if workspace is None:
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=qkv.device)
        if stream is not None and stream != torch.cuda.current_stream(qkv.device):
            workspace.record_stream(stream)  # the kernel runs on `stream`: keep the block alive until it finishes
    check(lib().atp_attn_core_bwd(qkv.data_ptr(), qkv.stride(0), ctx.data_ptr(), ctx.stride(0), lse.data_ptr(),
                                  dctx.data_ptr(), dctx.stride(0), T, seq, heads, head_dim, int(causal),
                                  dqkv.data_ptr(), dqkv.stride(0), workspace.data_ptr(), workspace.numel(),
                                  _stream(stream)))


# ------------------------------------------------------------------ linears
def _arr(struct_cls, items):
    arr = (struct_cls * len(items))()
    for i, it in enumerate(items):
        arr[i] = it
    return arr


def atp_linear_fwd(mesh: Mesh, colfirst: bool, per_rank: list[dict], M: int, K: int, N: int, chunks: int = 1,
                   stream=None):
    """per_rank: [{x, w, bias (or None), y}] — one dict per local rank (torch tensors)."""
    a = _arr(_abi.LinearFwdArgs, [_abi.LinearFwdArgs(d["x"].data_ptr(), d["w"].data_ptr(), _ptr(d.get("bias")),
                                                     d["y"].data_ptr()) for d in per_rank])
    f = lib().atp_linear_colfirst_fwd if colfirst else lib().atp_linear_rowfirst_fwd
    check(f(mesh.handle, a, M, K, N, chunks, _dt(per_rank[0]["x"]), _stream(stream)))


def atp_linear_bwd(mesh: Mesh, colfirst: bool, per_rank: list[dict], M: int, K: int, N: int, chunks: int = 1,
                   stream=None):
    """per_rank: [{x, w, dy, dx, dw (fp32), dbias (fp32 or None)}]."""
    a = _arr(_abi.LinearBwdArgs, [_abi.LinearBwdArgs(d["x"].data_ptr(), d["w"].data_ptr(), d["dy"].data_ptr(),
                                                     d["dx"].data_ptr(), _ptr(d.get("dw")), _ptr(d.get("dbias")))
                                  for d in per_rank])
    f = lib().atp_linear_colfirst_bwd if colfirst else lib().atp_linear_rowfirst_bwd
    check(f(mesh.handle, a, M, K, N, chunks, _dt(per_rank[0]["x"]), _stream(stream)))


# ------------------------------------------------------------------ layer buffers
def _attn_fwd(b):
    return _abi.AttnFwdArgs(b["x"].data_ptr(), b["wqkv"].data_ptr(), _ptr(b.get("bqkv")), b["wo"].data_ptr(),
                            _ptr(b.get("bo")), b["qkv"].data_ptr(), b["ctx"].data_ptr(), b["y1"].data_ptr())


def _mlp_fwd(b):
    return _abi.MlpFwdArgs(b["y1"].data_ptr(), b["w1"].data_ptr(), _ptr(b.get("b1")), b["w2"].data_ptr(),
                           _ptr(b.get("b2")), b["u"].data_ptr(), b["h"].data_ptr(), b["z"].data_ptr())


def _mlp_bwd(b):
    return _abi.MlpBwdArgs(b["y1"].data_ptr(), b["w1"].data_ptr(), b["w2"].data_ptr(), b["u"].data_ptr(),
                           b["h"].data_ptr(), b["dz"].data_ptr(), b["dy1"].data_ptr(), _ptr(b["dw1"]),
                           _ptr(b["db1"]), _ptr(b["dw2"]), _ptr(b["db2"]), b["ws_dh"].data_ptr())


def _attn_bwd(b):
    return _abi.AttnBwdArgs(b["x"].data_ptr(), b["wqkv"].data_ptr(), b["wo"].data_ptr(), b["ctx"].data_ptr(),
                            b["dy1"].data_ptr(), b["dx"].data_ptr(), _ptr(b["dwqkv"]), _ptr(b["dbqkv"]),
                            _ptr(b["dwo"]), _ptr(b["dbo"]), b["ws_dctx"].data_ptr(), b["ws_dqkv"].data_ptr())


def _dt(t) -> int:
    import torch

    return _abi.ATP_FP32 if t.dtype == torch.float32 else _abi.ATP_BF16


def _gen_block(name, shape, r0, nr, c0, nc, device, seed, bf16=True, host=False):
    """One block of a seeded global input (datagen): generated on the device, or
    with host=True on the host (numpy) and copied in (no device kernel besides the copy)."""
    import numpy as np
    import torch
    import datagen

    if not host:
        return datagen.torch_block(name, shape, r0, nr, c0, nc, device, seed=seed, bf16=bf16)
    cols = np.arange(c0, c0 + nc)
    v = (datagen.tensor(name, shape, seed=seed, bf16=bf16, cols=cols) if len(shape) == 1 else
         datagen.tensor(name, shape, seed=seed, bf16=bf16, rows=np.arange(r0, r0 + nr), cols=cols))
    # cast on the host (exact: the values are bf16-representable), then one H2D copy
    return torch.from_numpy(np.ascontiguousarray(v.reshape(nr, nc))).to(
        dtype=torch.bfloat16 if bf16 else torch.float32).to(device=device)


def alloc_layer_rank(d1: int, d2: int, rank: int, T: int, h: int, F: int, device, seed: int, with_bias: bool = True,
                     inputs: bool = True, fp32: bool = False, host_inputs: bool = False) -> dict:
    """Allocate one rank's layer buffers; fill inputs/weights from the seeded
    counter-based generator (datagen) directly on the device (host_inputs=True:
    on the host, then one copy).  fp32=True: the ATP_FP32 check mode (fp32
    storage, unrounded fp32 inputs)."""
    import torch
    import datagen

    w = layout.local_widths(d1, d2, h, F)
    hc, h1, q1, F1 = w["hc"], w["h1"], w["q1"], w["F1"]
    bf, f32 = (torch.float32 if fp32 else torch.bfloat16), torch.float32
    box = layout.shard_boxes(d1, d2, rank, T, h, F)
    shapes = datagen.layer_shapes(T, h, F)
    b = {}
    for name in ("x", "dz", "wqkv", "wo", "w1", "w2") + (("bqkv", "bo", "b1", "b2") if with_bias else ()):
        r0, nr, c0, nc = box[name]
        if inputs:
            t = _gen_block(name, shapes[name], r0, nr, c0, nc, device, seed, bf16=not fp32, host=host_inputs)
        else:
            t = torch.empty((nr, nc), dtype=bf, device=device)
        b[name] = t.reshape(-1) if name.startswith("b") else t
    E = lambda *s, dt=bf: torch.empty(s, dtype=dt, device=device)
    b.update(qkv=E(T, q1), ctx=E(T, h1), y1=E(T, hc), u=E(T, F1), h=E(T, F1), z=E(T, hc),
             dy1=E(T, hc), dx=E(T, hc), ws_dh=E(T, F1), ws_dctx=E(T, h1), ws_dqkv=E(T, q1),
             dwqkv=E(hc, q1, dt=f32), dbqkv=E(q1, dt=f32), dwo=E(h1, hc, dt=f32), dbo=E(hc, dt=f32),
             dw1=E(hc, F1, dt=f32), db1=E(F1, dt=f32), dw2=E(F1, hc, dt=f32), db2=E(hc, dt=f32))
    return b


def atp_attn_proj_fwd(mesh, bufs, T, h, heads, chunks=1, stream=None):
    a = _arr(_abi.AttnFwdArgs, [_attn_fwd(b) for b in bufs])
    check(lib().atp_attn_proj_fwd(mesh.handle, a, T, h, heads, chunks, _abi.ATP_CORE_SUM_QKV, _dt(bufs[0]["x"]),
                                  _stream(stream)))


def atp_attn_proj_bwd(mesh, bufs, T, h, heads, chunks=1, stream=None):
    a = _arr(_abi.AttnBwdArgs, [_attn_bwd(b) for b in bufs])
    check(lib().atp_attn_proj_bwd(mesh.handle, a, T, h, heads, chunks, _abi.ATP_CORE_SUM_QKV, _dt(bufs[0]["x"]),
                                  _stream(stream)))


def atp_mlp_fwd(mesh, bufs, T, h, F, chunks=1, stream=None):
    a = _arr(_abi.MlpFwdArgs, [_mlp_fwd(b) for b in bufs])
    check(lib().atp_mlp_fwd(mesh.handle, a, T, h, F, chunks, _dt(bufs[0]["y1"]), _stream(stream)))


def atp_mlp_bwd(mesh, bufs, T, h, F, chunks=1, stream=None):
    a = _arr(_abi.MlpBwdArgs, [_mlp_bwd(b) for b in bufs])
    check(lib().atp_mlp_bwd(mesh.handle, a, T, h, F, chunks, _dt(bufs[0]["y1"]), _stream(stream)))


class Graph:
    """A CUDA graph of libatp calls on one mesh (atp_graph_begin/end/launch):
    `Graph.capture(mesh, fn, stream)` runs `fn(stream)` once uncaptured
    (first-use setup), then captures it; calling the Graph replays it."""

    def __init__(self, handle):
        self.handle = handle

    @classmethod
    def capture(cls, mesh: "Mesh", fn, stream=None) -> "Graph":
        import torch

        st = stream if stream is not None else torch.cuda.current_stream()
        if st.cuda_stream == 0:
            raise AtpError("Graph.capture: needs a non-default stream (legacy stream 0 cannot be captured)")
        fn(st)
        st.synchronize()
        check(lib().atp_graph_begin(mesh.handle, st.cuda_stream))
        try:
            fn(st)
        finally:
            h = C.c_void_p()
            rc = lib().atp_graph_end(mesh.handle, st.cuda_stream, C.byref(h))
        check(rc)
        return cls(h.value)

    def __call__(self, stream=None) -> None:
        check(lib().atp_graph_launch(self.handle, _stream(stream)))

    def destroy(self) -> None:
        if self.handle:
            lib().atp_graph_destroy(self.handle)
            self.handle = None


class LayerCall:
    """Pre-marshalled argument array for repeated atp_layer_fwd_bwd calls (bench loop)."""

    def __init__(self, mesh, bufs, T, h, F, heads, chunks=1, backward=True):
        self.mesh = mesh
        self.args = _arr(_abi.LayerArgs, [_abi.LayerArgs(_attn_fwd(b), _mlp_fwd(b), _mlp_bwd(b), _attn_bwd(b))
                                          for b in bufs])
        self.dims = (T, h, F, heads, chunks, int(backward))
        self.dtype = _dt(bufs[0]["x"])
        self._f = lib().atp_layer_fwd_bwd

    def __call__(self, stream=None):
        T, h, F, heads, chunks, bwd = self.dims
        check(self._f(self.mesh.handle, self.args, T, h, F, heads, chunks, bwd, self.dtype, _stream(stream)))


def atp_layer_fwd_bwd(mesh, bufs, T, h, F, heads, chunks=1, backward=True, stream=None):
    LayerCall(mesh, bufs, T, h, F, heads, chunks, backward)(stream)


def alloc_layer_stack(d1: int, d2: int, rank: int, T: int, h: int, F: int, device, seed: int, n_layers: int,
                      **kw) -> list[dict]:
    """One rank's buffers of an n-layer stack (layer l's weights from seed + l):
    layer l+1's input x IS layer l's output z, and layer l's upstream gradient
    dz IS layer l+1's input gradient dx (atp_layer_stack_fwd_bwd's chaining)."""
    st = [alloc_layer_rank(d1, d2, rank, T, h, F, device, seed + l, **kw) for l in range(n_layers)]
    for l in range(1, n_layers):
        st[l]["x"] = st[l - 1]["z"]
    for l in range(n_layers - 1):
        st[l]["dz"] = st[l + 1]["dx"]
    return st


class LayerStackCall:
    """Pre-marshalled atp_layer_stack_fwd_bwd: stack[l][i] = layer l's buffers of local rank i."""

    def __init__(self, mesh, stack, T, h, F, heads, chunks=1):
        self.mesh = mesh
        self.n_layers = len(stack)
        self.args = _arr(_abi.LayerArgs, [_abi.LayerArgs(_attn_fwd(b), _mlp_fwd(b), _mlp_bwd(b), _attn_bwd(b))
                                          for layer in stack for b in layer])
        self.dims = (T, h, F, heads, chunks)
        self.dtype = _dt(stack[0][0]["x"])
        self._f = lib().atp_layer_stack_fwd_bwd

    def __call__(self, stream=None):
        T, h, F, heads, chunks = self.dims
        check(self._f(self.mesh.handle, self.args, self.n_layers, T, h, F, heads, chunks, self.dtype,
                      _stream(stream)))


# ------------------------------------------------------------------ workspace sizes
ATP_OP_MLP_BWD, ATP_OP_ATTN_BWD, ATP_OP_LAYER, ATP_OP_GPT_LAYER = 0, 1, 2, 3


def atp_workspace_size(op: int, d1: int, d2: int, T: int, h: int, F: int, heads: int = 0, seq: int = 0,
                       chunks: int = 1) -> list[int]:
    """Bytes of each caller-allocated workspace buffer of `op` (struct order; unused = 0)."""
    out = (C.c_size_t * 4)()
    check(lib().atp_workspace_size(op, d1, d2, T, h, F, heads, seq, chunks, out))
    return [int(v) for v in out]


# ------------------------------------------------------------------ full GPT layer
def gpt_boxes(d1: int, d2: int, rank: int, T: int, h: int, F: int) -> dict:
    """(row0, nrows, col0, ncols) of rank's shard of every global input (oracle/gpt.shard_gpt
    layout; bqkv is the whole d1 block: the GPU adds it on i2 == 0 before the reduce-scatter)."""
    box = layout.shard_boxes(d1, d2, rank, T, h, F)
    out = {k: box[k] for k in ("x", "dz", "wqkv", "bqkv", "wo", "bo", "w1", "b1", "w2", "b2")}
    for k in ("g1", "be1", "g2", "be2"):
        out[k] = box["bo"]
    return out


def alloc_gpt_rank(d1: int, d2: int, rank: int, T: int, h: int, F: int, heads: int, device, seed: int,
                   inputs: bool = True, host_inputs: bool = False) -> dict:
    """One rank's full-layer buffers (inputs from the seeded generator, on the
    device, or with host_inputs=True on the host and copied in)."""
    import torch
    import datagen

    hc, h1, q1, F1 = h // d2, h // d1, 3 * h // d1, F // d1
    ql, cl, hl = q1 // d2, h1 // d2, heads // (d1 * d2)
    shapes = datagen.gpt_shapes(T, h, F)
    b = {}
    for name, (r0, nr, c0, nc) in gpt_boxes(d1, d2, rank, T, h, F).items():
        t = (_gen_block(name, shapes[name], r0, nr, c0, nc, device, seed, host=host_inputs) if inputs
             else torch.empty((nr, nc), dtype=torch.bfloat16, device=device))
        b[name] = t.reshape(-1) if len(shapes[name]) == 1 else t
    bf, f32 = torch.bfloat16, torch.float32
    E = lambda *s, dt=bf: torch.empty(s, dtype=dt, device=device)
    b.update(a=E(T, hc), sv1=E(T, 2, dt=f32), qkv=E(T, ql), ctx_loc=E(T, cl), lse=E(T * hl, dt=f32), ctx=E(T, h1),
             y1=E(T, hc), bn=E(T, hc), sv2=E(T, 2, dt=f32), u=E(T, F1), h=E(T, F1), z=E(T, hc), dx=E(T, hc),
             dwqkv=E(hc, q1, dt=f32), dbqkv=E(q1, dt=f32), dwo=E(h1, hc, dt=f32), dbo=E(hc, dt=f32),
             dw1=E(hc, F1, dt=f32), db1=E(F1, dt=f32), dw2=E(F1, hc, dt=f32), db2=E(hc, dt=f32),
             dg1=E(hc, dt=f32), dbe1=E(hc, dt=f32), dg2=E(hc, dt=f32), dbe2=E(hc, dt=f32))
    return b


class GptCall:
    """Pre-marshalled atp_gpt_layer_fwd_bwd call (one args entry per local rank) with its workspace."""

    def __init__(self, mesh, bufs, T, h, F, heads, seq, chunks=1, causal=True):
        import torch

        self.mesh = mesh
        self.args = _arr(_abi.GptArgs, [_abi.GptArgs(*[bb[n].data_ptr() for n in _abi.GPT_FIELDS]) for bb in bufs])
        self.dims = (T, h, F, heads, seq, chunks, int(causal))
        per = lib().atp_gpt_workspace(mesh.d1, mesh.d2, T, h, F, heads, seq, chunks)
        self.ws = torch.empty(per * len(bufs), dtype=torch.uint8, device=bufs[0]["x"].device)
        self._f = lib().atp_gpt_layer_fwd_bwd

    def __call__(self, stream=None):
        T, h, F, heads, seq, chunks, causal = self.dims
        check(self._f(self.mesh.handle, self.args, T, h, F, heads, seq, chunks, causal, self.ws.data_ptr(),
                      self.ws.numel(), _stream(stream)))


# ------------------------------------------------------------------ cost model
@dataclass
class HcmLayer:
    ranks: int
    p2p_gbps: float
    group_gbps: float


def _hcm(layers) -> _abi.Hcm:
    H = _abi.Hcm()
    H.n_layers = len(layers)
    for j, l in enumerate(layers):
        H.ranks[j] = l.ranks
        H.p2p_gbps[j] = l.p2p_gbps
        H.group_gbps[j] = l.group_gbps
    return H


def atp_effective_bandwidth(layers, d1: int, d2: int):
    b1, b2 = C.c_double(), C.c_double()
    check(lib().atp_effective_bandwidth(C.byref(_hcm(layers)), d1, d2, C.byref(b1), C.byref(b2)))
    return (b1.value if d1 > 1 else None), (b2.value if d2 > 1 else None)


def atp_search(layers, L=1, b=4, s=2048, h=4096, heads=32, bytes_per_elem=2, calibration: dict | None = None):
    """Ranked plan: list of dicts (ascending t_comm) and the chosen (d1, d2)."""
    n = 1
    for l in layers:
        n *= l.ranks
    m = _abi.Model(L, b, s, h, heads, bytes_per_elem)
    cal = None
    if calibration:
        cal = _abi.Calib()
        cal.n = len(calibration)
        for i, ((d1, d2), (b1, b2)) in enumerate(calibration.items()):
            cal.d1[i], cal.d2[i] = d1, d2
            cal.b1[i] = b1 if b1 else 0.0
            cal.b2[i] = b2 if b2 else 0.0
    plan = _abi.Plan()
    check(lib().atp_search(C.byref(_hcm(layers)), C.byref(m), n, C.byref(cal) if cal else None, C.byref(plan)))
    ranked = []
    for i in range(plan.n_ranked):
        c = plan.ranked[i]
        ranked.append({"d1": c.d1, "d2": c.d2, "b1_prime": c.b1_prime, "b2_prime": c.b2_prime, "b1": c.b1,
                       "b2": c.b2, "t_f": list(c.t_f), "t_comm": c.t_comm, "calibrated": bool(c.calibrated)})
    rejected = [(plan.rejected_d1[i], plan.rejected_d2[i]) for i in range(plan.n_rejected)]
    return {"ranked": ranked, "chosen": (ranked[0]["d1"], ranked[0]["d2"]), "rejected": rejected}


def atp_comm_volume(d1, d2, T, h, F=None, chunks=1):
    F = 4 * h if F is None else F
    n = C.c_int()
    e1, e2 = C.c_int64(), C.c_int64()
    check(lib().atp_comm_volume(d1, d2, T, h, F, chunks, None, 0, C.byref(n), C.byref(e1), C.byref(e2)))
    calls = (_abi.Call * max(n.value, 1))()
    check(lib().atp_comm_volume(d1, d2, T, h, F, chunks, calls, n.value, C.byref(n), C.byref(e1), C.byref(e2)))
    names = ["qkv", "out", "fc1", "fc2"]
    out = [(("fwd", "bwd")[c.phase], names[c.block], c.dim, c.p, c.elems) for c in calls[:n.value]]
    return out, e1.value, e2.value


def atp_probe_allreduce(mesh: Mesh, dim: int, buf, msg_bytes: int, iters: int = 20):
    bus, alg, sec = C.c_double(), C.c_double(), C.c_double()
    check(lib().atp_probe_allreduce(mesh.handle, dim, msg_bytes, iters, buf.data_ptr(), C.byref(bus),
                                    C.byref(alg), C.byref(sec)))
    return {"busbw_gbps": bus.value, "algbw_gbps": alg.value, "seconds": sec.value}


def atp_probe_hcm(mesh: Mesh, scratch, msg_bytes=(64 << 20, 256 << 20), calib_bytes=16 << 20, iters: int = 10):
    """S1 probe on a distributed mesh of all ranks (collective).  Returns
    (hcm layers, p2p matrix [N][N] GB/s, calibration {(d1, d2): (B1, B2)})."""
    n = mesh.d1 * mesh.d2
    sizes = (C.c_size_t * len(msg_bytes))(*msg_bytes)
    H = _abi.Hcm()
    pm = (C.c_double * (n * n))()
    cal = _abi.Calib()
    check(lib().atp_probe_hcm(mesh.handle, sizes, len(msg_bytes), calib_bytes, iters, scratch.data_ptr(),
                              C.byref(H), pm, C.byref(cal)))
    layers = [HcmLayer(H.ranks[j], H.p2p_gbps[j], H.group_gbps[j]) for j in range(H.n_layers)]
    matrix = [[pm[i * n + j] for j in range(n)] for i in range(n)]
    calib = {(cal.d1[k], cal.d2[k]): (cal.b1[k] or None, cal.b2[k] or None) for k in range(cal.n)}
    return layers, matrix, calib


def atp_overlap_estimate(stages, chunks: int, mode: str = "signalled"):
    """stages = [(comp, dw, comm), ...] -> (makespan, exposed) of the chunk pipeline model."""
    n = len(stages)
    arr = lambda i: (C.c_double * max(n, 1))(*[s[i] for s in stages])
    mk, ex = C.c_double(), C.c_double()
    check(lib().atp_overlap_estimate(n, arr(0), arr(1), arr(2), chunks, 0 if mode == "signalled" else 1,
                                     C.byref(mk), C.byref(ex)))
    return mk.value, ex.value


def atp_layer_stages(T, h, F, d1, d2, compute_ms, busbw_gbps, bytes_per_elem=2):
    """[(comp_ms, dw_ms, comm_ms)] x 8 stages of one layer fwd+bwd (libatp's planner decomposition)."""
    a, b, c = (C.c_double * 8)(), (C.c_double * 8)(), (C.c_double * 8)()
    check(lib().atp_layer_stages(d1, d2, T, h, F, bytes_per_elem, compute_ms, busbw_gbps, a, b, c))
    return [(a[i], b[i], c[i]) for i in range(8)]


def atp_plan_chunks(T, h, F, d1, d2, compute_ms_by_c: dict, busbw_gbps: float, mode: str = "signalled",
                    bytes_per_elem: int = 2):
    """Chunk count with the smallest predicted step (libatp atp_plan_chunks).
    Returns (chosen c, {c: (makespan_ms, exposed_ms)})."""
    cs = sorted(compute_ms_by_c)
    n = len(cs)
    ch = (C.c_int * n)(*cs)
    cm = (C.c_double * n)(*[float(compute_ms_by_c[c]) for c in cs])
    mk, ex, chosen = (C.c_double * n)(), (C.c_double * n)(), C.c_int()
    check(lib().atp_plan_chunks(d1, d2, T, h, F, bytes_per_elem, n, ch, cm, busbw_gbps,
                                0 if mode == "signalled" else 1, C.byref(chosen), mk, ex))
    return chosen.value, {c: (mk[i], ex[i]) for i, c in enumerate(cs)}
