"""ctypes declarations of include/atp.h (argument marshalling only).

Loading fails loudly if ``libatp.so`` is missing: there is no CPU or PyTorch
fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libatp.so")

ATP_OK, ATP_ERR_INVALID, ATP_ERR_SHAPE, ATP_ERR_CUDA, ATP_ERR_NCCL, ATP_ERR_EMPTY, ATP_ERR_UNSUPPORTED = range(7)
STATUS_NAMES = ["ATP_OK", "ATP_ERR_INVALID", "ATP_ERR_SHAPE", "ATP_ERR_CUDA", "ATP_ERR_NCCL", "ATP_ERR_EMPTY",
                "ATP_ERR_UNSUPPORTED"]
ATP_BF16 = 0
ATP_FP32 = 1
ATP_CORE_SUM_QKV = 0
ATP_MAX_HCM_LAYERS = 8
ATP_MAX_PLAN = 64

vp = C.c_void_p
fp = C.POINTER(C.c_float)
i64 = C.c_int64


class AtpError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else status}: {msg}")
        self.status = status


class LinearFwdArgs(C.Structure):
    _fields_ = [("x", vp), ("w", vp), ("bias", vp), ("y", vp)]


class LinearBwdArgs(C.Structure):
    _fields_ = [("x", vp), ("w", vp), ("dy", vp), ("dx", vp), ("dw", vp), ("dbias", vp)]


class MlpFwdArgs(C.Structure):
    _fields_ = [("x", vp), ("w1", vp), ("b1", vp), ("w2", vp), ("b2", vp), ("u", vp), ("h_act", vp), ("z", vp)]


class MlpBwdArgs(C.Structure):
    _fields_ = [("x", vp), ("w1", vp), ("w2", vp), ("u", vp), ("h_act", vp), ("dz", vp), ("dx", vp),
                ("dw1", vp), ("db1", vp), ("dw2", vp), ("db2", vp), ("ws_dh", vp)]


class AttnFwdArgs(C.Structure):
    _fields_ = [("x", vp), ("wqkv", vp), ("bqkv", vp), ("wo", vp), ("bo", vp), ("qkv", vp), ("ctx", vp), ("y", vp)]


class AttnBwdArgs(C.Structure):
    _fields_ = [("x", vp), ("wqkv", vp), ("wo", vp), ("ctx", vp), ("dy", vp), ("dx", vp), ("dwqkv", vp),
                ("dbqkv", vp), ("dwo", vp), ("dbo", vp), ("ws_dctx", vp), ("ws_dqkv", vp)]


class LayerArgs(C.Structure):
    _fields_ = [("attn", AttnFwdArgs), ("mlp", MlpFwdArgs), ("mlp_b", MlpBwdArgs), ("attn_b", AttnBwdArgs)]


class Hcm(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("ranks", C.c_int * ATP_MAX_HCM_LAYERS),
                ("p2p_gbps", C.c_double * ATP_MAX_HCM_LAYERS), ("group_gbps", C.c_double * ATP_MAX_HCM_LAYERS)]


class Model(C.Structure):
    _fields_ = [("L", i64), ("b", i64), ("s", i64), ("h", i64), ("heads", i64), ("bytes_per_elem", i64)]


class Calib(C.Structure):
    _fields_ = [("n", C.c_int), ("d1", C.c_int * ATP_MAX_PLAN), ("d2", C.c_int * ATP_MAX_PLAN),
                ("b1", C.c_double * ATP_MAX_PLAN), ("b2", C.c_double * ATP_MAX_PLAN)]


class Cost(C.Structure):
    _fields_ = [("d1", C.c_int), ("d2", C.c_int), ("b1_prime", C.c_double), ("b2_prime", C.c_double),
                ("b1", C.c_double), ("b2", C.c_double), ("t_f", C.c_double * 4), ("t_comm", C.c_double),
                ("calibrated", C.c_int)]


class Plan(C.Structure):
    _fields_ = [("n_ranked", C.c_int), ("ranked", Cost * ATP_MAX_PLAN), ("chosen", C.c_int),
                ("n_rejected", C.c_int), ("rejected_d1", C.c_int * ATP_MAX_PLAN),
                ("rejected_d2", C.c_int * ATP_MAX_PLAN)]


GPT_FIELDS = ("x", "dz", "g1", "be1", "g2", "be2", "wqkv", "bqkv", "wo", "bo", "w1", "b1", "w2", "b2",
              "a", "sv1", "qkv", "ctx_loc", "lse", "ctx", "y1", "bn", "sv2", "u", "h", "z", "dx",
              "dwqkv", "dbqkv", "dwo", "dbo", "dw1", "db1", "dw2", "db2", "dg1", "dbe1", "dg2", "dbe2")


class GptArgs(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in GPT_FIELDS]


class Profile(C.Structure):
    _fields_ = [("launches", i64 * 4), ("ms", C.c_double * 4), ("flops", C.c_double * 4), ("bytes", C.c_double * 4)]


class TraceRec(C.Structure):
    _fields_ = [("cls", C.c_int), ("stream", C.c_int), ("kind", C.c_int), ("sub", C.c_int), ("t0_ms", C.c_double),
                ("t1_ms", C.c_double)]


class Call(C.Structure):
    _fields_ = [("phase", C.c_int), ("block", C.c_int), ("dim", C.c_int), ("p", C.c_int), ("elems", i64)]


# name -> (restype, argtypes)
SIGNATURES = {
    "atp_last_error": (C.c_char_p, []),
    "atp_version": (C.c_char_p, []),
    "atp_get_unique_id": (C.c_int, [C.c_char_p]),
    "atp_mesh_init": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_int, C.POINTER(vp)]),
    "atp_vmesh_init": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(vp)]),
    "atp_mesh_init_local": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]),
    "atp_mesh_destroy": (C.c_int, [vp]),
    "atp_mesh_coords": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "atp_mesh_dims": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "atp_mesh_groups": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)]),
    "atp_mesh_set_gemm_ctas": (C.c_int, [vp, C.c_int]),
    "atp_mesh_set_gating": (C.c_int, [vp, C.c_int]),
    "atp_mesh_enable_fused_ar": (C.c_int, [vp, C.c_size_t]),
    "atp_mesh_set_comm_enabled": (C.c_int, [vp, C.c_int]),
    "atp_debug_counters": (C.c_int, [vp, C.c_int, C.POINTER(C.c_uint32), C.c_int]),
    "atp_profile_begin": (C.c_int, [vp]),
    "atp_profile_end": (C.c_int, [vp, C.POINTER(Profile)]),
    "atp_profile_trace": (C.c_int, [vp, C.POINTER(TraceRec), C.c_int, C.POINTER(C.c_int)]),
    "atp_launch_count": (C.c_int, [C.POINTER(C.c_uint64)]),
    "atp_graph_begin": (C.c_int, [vp, vp]),
    "atp_graph_end": (C.c_int, [vp, vp, C.POINTER(vp)]),
    "atp_graph_launch": (C.c_int, [vp, vp]),
    "atp_graph_destroy": (C.c_int, [vp]),
    "atp_attn_core_fwd": (C.c_int, [vp, i64, i64, i64, C.c_int, C.c_int, C.c_int, vp, i64, vp, vp]),
    "atp_attn_core_bwd": (C.c_int, [vp, i64, vp, i64, vp, vp, i64, i64, i64, C.c_int, C.c_int, C.c_int, vp, i64,
                                    vp, C.c_size_t, vp]),
    "atp_attn_core_workspace": (C.c_size_t, [i64, C.c_int]),
    "atp_mesh_init_from_comms": (C.c_int, [C.c_int, C.c_int, C.c_int, vp, vp, C.c_int, C.POINTER(vp)]),
    "atp_workspace_size": (C.c_int, [C.c_int, C.c_int, C.c_int, i64, i64, i64, i64, i64, C.c_int,
                                     C.POINTER(C.c_size_t)]),
    "atp_gpt_workspace": (C.c_size_t, [C.c_int, C.c_int, i64, i64, i64, i64, i64, C.c_int]),
    "atp_gpt_layer_fwd_bwd": (C.c_int, [vp, C.POINTER(GptArgs), i64, i64, i64, i64, i64, C.c_int, C.c_int, vp,
                                        C.c_size_t, vp]),
    "atp_gemm": (C.c_int, [vp, i64, C.c_int, vp, i64, C.c_int, vp, i64, C.c_int, vp, i64, i64, i64, C.c_int, vp]),
    "atp_linear_colfirst_fwd": (C.c_int, [vp, C.POINTER(LinearFwdArgs), i64, i64, i64, C.c_int, C.c_int, vp]),
    "atp_linear_rowfirst_fwd": (C.c_int, [vp, C.POINTER(LinearFwdArgs), i64, i64, i64, C.c_int, C.c_int, vp]),
    "atp_linear_colfirst_bwd": (C.c_int, [vp, C.POINTER(LinearBwdArgs), i64, i64, i64, C.c_int, C.c_int, vp]),
    "atp_linear_rowfirst_bwd": (C.c_int, [vp, C.POINTER(LinearBwdArgs), i64, i64, i64, C.c_int, C.c_int, vp]),
    "atp_mlp_fwd": (C.c_int, [vp, C.POINTER(MlpFwdArgs), i64, i64, i64, C.c_int, C.c_int, vp]),
    "atp_mlp_bwd": (C.c_int, [vp, C.POINTER(MlpBwdArgs), i64, i64, i64, C.c_int, C.c_int, vp]),
    "atp_attn_proj_fwd": (C.c_int, [vp, C.POINTER(AttnFwdArgs), i64, i64, i64, C.c_int, C.c_int, C.c_int, vp]),
    "atp_attn_proj_bwd": (C.c_int, [vp, C.POINTER(AttnBwdArgs), i64, i64, i64, C.c_int, C.c_int, C.c_int, vp]),
    "atp_layer_fwd_bwd": (C.c_int, [vp, C.POINTER(LayerArgs), i64, i64, i64, i64, C.c_int, C.c_int, C.c_int, vp]),
    "atp_layer_stack_fwd_bwd": (C.c_int, [vp, C.POINTER(LayerArgs), C.c_int, i64, i64, i64, i64, C.c_int, C.c_int,
                                          vp]),
    "atp_search": (C.c_int, [C.POINTER(Hcm), C.POINTER(Model), C.c_int, C.POINTER(Calib), C.POINTER(Plan)]),
    "atp_effective_bandwidth": (C.c_int, [C.POINTER(Hcm), C.c_int, C.c_int, C.POINTER(C.c_double),
                                          C.POINTER(C.c_double)]),
    "atp_comm_volume": (C.c_int, [C.c_int, C.c_int, i64, i64, i64, C.c_int, C.POINTER(Call), C.c_int,
                                  C.POINTER(C.c_int), C.POINTER(i64), C.POINTER(i64)]),
    "atp_overlap_estimate": (C.c_int, [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                       C.POINTER(C.c_double), C.c_int, C.c_int, C.POINTER(C.c_double),
                                       C.POINTER(C.c_double)]),
    "atp_layer_stages": (C.c_int, [C.c_int, C.c_int, i64, i64, i64, C.c_int, C.c_double, C.c_double,
                                   C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "atp_plan_chunks": (C.c_int, [C.c_int, C.c_int, i64, i64, i64, C.c_int, C.c_int, C.POINTER(C.c_int),
                                  C.POINTER(C.c_double), C.c_double, C.c_int, C.POINTER(C.c_int),
                                  C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "atp_probe_hcm": (C.c_int, [vp, C.POINTER(C.c_size_t), C.c_int, C.c_size_t, C.c_int, vp, C.POINTER(Hcm),
                                C.POINTER(C.c_double), C.POINTER(Calib)]),
    "atp_probe_allreduce": (C.c_int, [vp, C.c_int, C.c_size_t, C.c_int, vp, C.POINTER(C.c_double),
                                      C.POINTER(C.c_double), C.POINTER(C.c_double)]),
}

_lib = None


def lib():
    """Load libatp.so (built by ``paper_2301_08658_b200.build``); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libatp.so not built ({LIB_PATH}); run `python -m paper_2301_08658_b200.build`."
                               " There is no fallback implementation.")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != ATP_OK:
        raise AtpError(status, lib().atp_last_error().decode(errors="replace"))
