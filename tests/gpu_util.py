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


def tile_rel_max(got, ref, tile=(128, 256)):
    """Largest relative Frobenius error over the [tile] blocks of a 2-D tensor
    (1-D tensors: blocks of tile[1] elements; ragged edge blocks included).
    A whole-tensor relF hides a wrong tile in a large output (one 128x256 tile
    of an 8192x16384 tensor moves the global relF by ~0.02 at most); this
    bound does not."""
    a = np.asarray(got, dtype=np.float64)
    b = np.asarray(ref, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError(f"shape {a.shape} != {b.shape}")
    if a.ndim == 1:
        a, b, tile = a[None, :], b[None, :], (1, tile[1])
    tr, tc = tile
    R, Cn = a.shape
    pr, pc = (-R) % tr, (-Cn) % tc
    d = np.pad(a - b, ((0, pr), (0, pc)))
    r = np.pad(b, ((0, pr), (0, pc)))
    nr, nc = d.shape[0] // tr, d.shape[1] // tc
    num = np.einsum("ijkl,ijkl->ik", d.reshape(nr, tr, nc, tc), d.reshape(nr, tr, nc, tc))
    den = np.einsum("ijkl,ijkl->ik", r.reshape(nr, tr, nc, tc), r.reshape(nr, tr, nc, tc))
    return float(np.sqrt(num / np.maximum(den, 1e-60)).max())


def assert_close(name, got, ref, tol, tile=(128, 256)):
    """Every element finite, global relF <= tol and every tile's relF <= tol."""
    g = np.asarray(got, dtype=np.float64)
    assert np.isfinite(g).all(), (name, "non-finite elements (unwritten output?)")
    e = rel(g, ref)
    assert e <= tol, (name, "global relF", e)
    t = tile_rel_max(g, ref, tile)
    assert t <= tol, (name, "worst tile relF", t)
    return e, t
