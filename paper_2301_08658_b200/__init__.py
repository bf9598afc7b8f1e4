"""B200-native ATP (Adaptive Tensor Parallelism, arXiv 2301.08658) hot path.

The product is ``libatp.so`` (C ABI, include/atp.h): tcgen05/TMEM/TMA GEMMs,
HBM-bound epilogue kernels, the chunked dual-stream pipeline over NCCL, and
the Eq. 2-4 mesh search.  This package is a thin ctypes binding to it.
"""
from .api import (  # noqa: F401
    Graph, HcmLayer, LayerCall, LayerStackCall, Mesh, alloc_layer_rank, alloc_layer_stack, atp_attn_proj_bwd, atp_attn_proj_fwd, atp_comm_volume,
    GptCall, alloc_gpt_rank, atp_attn_core_bwd, atp_attn_core_fwd, atp_effective_bandwidth, atp_gemm, atp_get_unique_id, atp_layer_fwd_bwd, atp_linear_bwd, atp_linear_fwd,
    atp_mesh_groups, atp_mlp_bwd, atp_mlp_fwd, atp_overlap_estimate, atp_probe_allreduce, atp_probe_hcm,
    atp_search, atp_layer_stages, atp_plan_chunks,
)
from ._abi import AtpError, LIB_PATH  # noqa: F401
