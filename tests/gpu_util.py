"""Helpers for the -m gpu tests (oracle side: numpy; GPU side: libatp via the binding)."""
import numpy as np

import datagen
from oracle import layer as olayer


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def to_np(t):
    import torch

    return t.detach().to(torch.float32).cpu().numpy().astype(np.float64)


def oracle_layer(T, h, F, heads, d1, d2, chunks, seed):
    """Oracle per-rank shards of every forward/backward tensor (fp64)."""
    g = {k: v.astype(np.float64) for k, v in datagen.layer_globals(T, h, F, seed=seed).items()}
    sh, fw, bw, log = olayer.run_layer(g, d1, d2, heads, chunks)
    return g, sh, fw, bw, log


def oracle_layer_fp32(T, h, F, heads, d1, d2, chunks, seed):
    """Oracle on unrounded fp32 inputs (the ATP_FP32 check mode's values)."""
    g = {k: v.astype(np.float64) for k, v in datagen.layer_globals(T, h, F, seed=seed, bf16=False).items()}
    sh, fw, bw, log = olayer.run_layer(g, d1, d2, heads, chunks)
    return g, sh, fw, bw, log


# GPU buffer name -> oracle (dict, key)
FWD_MAP = {"qkv": "qkv", "ctx": "ctx", "y1": "y1", "u": "u", "h": "h", "z": "z"}
BWD_MAP = {"dy1": "dy1", "dx": "dx", "dwqkv": "dwqkv", "dbqkv": "dbqkv", "dwo": "dwo", "dbo": "dbo",
           "dw1": "dw1", "db1": "db1", "dw2": "dw2", "db2": "db2"}
