"""Seeded, counter-based synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no GEMM, no reduction, no
sharding rule); it only maps ``(seed, tensor_id, flat global index)`` to a
value, so that any sub-block of a global tensor (one rank's shard, a few sampled
rows) can be generated independently and identically on either side.

Generator (SURVEY.md §8(d) "Synthetic inputs"):
    z     = splitmix64(seed XOR (tensor_id << 40) XOR flat_index)
    u     = (z >> 40) / 2**24                  in [0, 1)
    value = scale * (2u - 1)                    uniform in [-scale, scale)
    then rounded once to bf16 (round-to-nearest-even) when ``bf16=True``.

Scales: activations and upstream gradients have sigma 1 (scale sqrt(3)),
weights sigma 0.02 (scale 0.02*sqrt(3), GPT init), biases uniform +-0.02.
The paper names no value statistics (§5 P:375 gives only shapes and
FP16); these distributions are a stated choice, see DESIGN.md "Input recipe".
"""
from __future__ import annotations

import math

import numpy as np

BASE_SEED = 2301

# Fixed tensor-id table: every global tensor of one layer gets its own stream.
TENSOR_IDS = {
    "x": 1, "wqkv": 2, "bqkv": 3, "wo": 4, "bo": 5,
    "w1": 6, "b1": 7, "w2": 8, "b2": 9, "dz": 10,
    # full GPT layer (LayerNorm gamma / beta)
    "g1": 11, "be1": 12, "g2": 13, "be2": 14,
    # stand-alone linear tests
    "lin_x": 20, "lin_w": 21, "lin_b": 22, "lin_dy": 23,
}

ACT_SCALE = math.sqrt(3.0)
WEIGHT_SCALE = 0.02 * math.sqrt(3.0)
BIAS_SCALE = 0.02
GAMMA_SCALE = 0.1   # LayerNorm gamma = 1 + uniform(+-0.1) (never exactly the identity)

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def default_offset(name: str) -> float:
    return 1.0 if name in ("g1", "g2") else 0.0


def default_scale(name: str) -> float:
    if name in ("g1", "g2"):
        return GAMMA_SCALE
    if name in ("x", "dz", "lin_x", "lin_dy"):
        return ACT_SCALE
    if name.startswith("b") or name == "lin_b":
        return BIAS_SCALE
    return WEIGHT_SCALE


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def round_bf16(a: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bf16 (ties to even); returns float32."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    u = (u + np.uint64(0x7FFF) + lsb) & np.uint64(0xFFFF0000)
    return u.astype(np.uint32).view(np.float32)


def uniform_block(tensor_id: int, shape_global, rows, cols, scale: float,
                  seed: int = BASE_SEED, bf16: bool = True, offset: float = 0.0) -> np.ndarray:
    """Values of the global 2-D tensor ``[shape_global]`` at ``rows x cols``.

    ``rows``/``cols`` are ``range``/``slice``-like (start, stop) pairs or index
    arrays. Returns float32 (bf16-representable when ``bf16``).
    """
    n_rows, n_cols = shape_global
    r = np.asarray(rows, dtype=np.uint64).reshape(-1, 1)
    c = np.asarray(cols, dtype=np.uint64).reshape(1, -1)
    idx = r * np.uint64(n_cols) + c
    key = np.uint64(seed) ^ (np.uint64(tensor_id) << np.uint64(40))
    z = _splitmix64(idx ^ key)
    u = (z >> np.uint64(40)).astype(np.float64) / float(1 << 24)
    v = (offset + scale * (2.0 * u - 1.0)).astype(np.float32)
    return round_bf16(v) if bf16 else v


def tensor(name: str, shape, seed: int = BASE_SEED, bf16: bool = True,
           rows=None, cols=None, scale: float | None = None) -> np.ndarray:
    """Global tensor ``name`` of ``shape`` (1-D or 2-D), or a row/col sub-block."""
    tid = TENSOR_IDS[name]
    sc = default_scale(name) if scale is None else scale
    off = default_offset(name)
    if len(shape) == 1:
        (n,) = shape
        c = np.arange(n) if cols is None else np.asarray(cols)
        return uniform_block(tid, (1, n), [0], c, sc, seed, bf16, off).reshape(-1)
    nr, nc = shape
    r = np.arange(nr) if rows is None else np.asarray(rows)
    c = np.arange(nc) if cols is None else np.asarray(cols)
    if len(r) * len(c) < (1 << 22):
        return uniform_block(tid, (nr, nc), r, c, sc, seed, bf16, off)
    # large tensors: row blocks on a thread pool (numpy's integer ufuncs release the GIL)
    import os
    from concurrent.futures import ThreadPoolExecutor

    out = np.empty((len(r), len(c)), dtype=np.float32)
    step = max(1, (1 << 20) // max(1, len(c)))

    def fill(i0):
        out[i0:i0 + step] = uniform_block(tid, (nr, nc), r[i0:i0 + step], c, sc, seed, bf16, off)

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
        list(ex.map(fill, range(0, len(r), step)))
    return out


def layer_shapes(T: int, h: int, F: int) -> dict:
    """Global shapes of the layer's tensors in math orientation W[in, out]."""
    return {
        "x": (T, h), "wqkv": (h, 3 * h), "bqkv": (3 * h,), "wo": (h, h), "bo": (h,),
        "w1": (h, F), "b1": (F,), "w2": (F, h), "b2": (h,), "dz": (T, h),
    }


def gpt_shapes(T: int, h: int, F: int) -> dict:
    """Global shapes of the full GPT layer: the linear block plus LayerNorm gamma/beta."""
    s = layer_shapes(T, h, F)
    s.update({"g1": (h,), "be1": (h,), "g2": (h,), "be2": (h,)})
    return s


def gpt_globals(T: int, h: int, F: int, seed: int = BASE_SEED, bf16: bool = True) -> dict:
    return {k: tensor(k, s, seed, bf16) for k, s in gpt_shapes(T, h, F).items()}


def layer_globals(T: int, h: int, F: int, seed: int = BASE_SEED, bf16: bool = True) -> dict:
    """All global tensors of one layer (small configs only: materialises everything)."""
    return {k: tensor(k, s, seed, bf16) for k, s in layer_shapes(T, h, F).items()}


# ---------------------------------------------------------------------------
# Device-side twin (same counter-based stream, generated directly in HBM so the
# full-size bench does not push gigabytes through numpy).  Plain torch integer
# ops; no method arithmetic.
# ---------------------------------------------------------------------------
def _to_i64(v: int) -> int:
    v &= 0xFFFFFFFFFFFFFFFF
    return v - (1 << 64) if v >= (1 << 63) else v


def torch_block(name: str, shape_global, row0: int, nrows: int, col0: int, ncols: int,
                device, seed: int = BASE_SEED, scale: float | None = None, bf16: bool = True):
    """Torch tensor equal to ``tensor(name, shape_global, bf16=bf16)[row0:row0+nrows, col0:col0+ncols]``
    (bf16 dtype when ``bf16``, else the unrounded float32 values)."""
    import torch

    tid = TENSOR_IDS[name]
    sc = default_scale(name) if scale is None else scale
    if len(shape_global) == 1:
        n_cols = shape_global[0]
    else:
        n_cols = shape_global[1]
    key = _to_i64(seed ^ (tid << 40))
    out = torch.empty((nrows, ncols), dtype=torch.bfloat16 if bf16 else torch.float32, device=device)
    step = max(1, (1 << 24) // max(ncols, 1))
    c = torch.arange(col0, col0 + ncols, device=device, dtype=torch.int64).view(1, -1)
    for r0 in range(0, nrows, step):
        rr = min(step, nrows - r0)
        r = torch.arange(row0 + r0, row0 + r0 + rr, device=device, dtype=torch.int64).view(-1, 1)
        x = (r * n_cols + c) ^ key
        z = x + _to_i64(0x9E3779B97F4A7C15)
        z = (z ^ _lsr(z, 30)) * _to_i64(0xBF58476D1CE4E5B9)
        z = (z ^ _lsr(z, 27)) * _to_i64(0x94D049BB133111EB)
        z = z ^ _lsr(z, 31)
        u = _lsr(z, 40).to(torch.float64) / float(1 << 24)
        v = (default_offset(name) + sc * (2.0 * u - 1.0)).to(torch.float32)
        out[r0:r0 + rr] = v.to(torch.bfloat16) if bf16 else v  # torch's f32->bf16 cast is RNE
    return out


def _lsr(z, s: int):
    """Logical right shift of int64 viewed as uint64."""
    import torch

    return (z >> s) & ((1 << (64 - s)) - 1)
