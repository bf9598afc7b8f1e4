"""Benchmark of the ATP linear block (attention projections + MLP, fwd+bwd) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl atp|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1, one rank per GPU)

One step = one GPT layer's linear block forward + backward on DeviceMesh(d1, d2)
(F3..F12, B1..B6 of SURVEY.md §8(a)) through libatp's C ABI.  Prints ONE JSON
line on rank 0.  Timing: W untimed warm-up steps, then K steps bracketed by
barrier + cudaDeviceSynchronize, CUDA events on the launching stream, max over
ranks.  The working set (weights + activations, GBs) is far larger than the
126 MB L2, so no explicit flush is done (stated in `config`).

Workload per N (BASELINE.json configs; override with --hidden/--heads):
  N = 1      cfg 5 shape h=12288, a=96 (the largest single-GPU configuration)
  N = 2, 4   cfg 2, h=4096, a=32
  N = 8      cfg 4, h=5120, a=40 (the north_star target) on the atp_search mesh
All: b=4, s=2048 (T=8192 tokens), F=4h, bf16.

At N > 1 (default) the HCM probe (atp_probe_hcm, §3.4 / P:482) runs first: its
calibrated bandwidths feed atp_search (the mesh) and its bus bandwidth feeds the
chunk planner (atp_plan_chunks, §4.1), together with the measured compute-side
time of each candidate chunk count.

Extra passes after the timed region (reported, never mixed into `value`):
  * comm-disabled twin  -> exposed_comm_ms = t - t(no all-reduce)       (N > 1)
  * Megatron-style baseline: the same library at DeviceMesh(N,1), 1 chunk (N > 1)
  * CUPTI kernel trace of the same graph-launched step -> roofline (GEMM time
    and share of the step), cross-checked by per-launch CUDA events
  * e2e pass            -> same step through the public API with the step's
                           inputs (X, dZ) copied H2D from pinned memory and its
                           result (the bias gradients) read D2H each step
  * cpu_baseline        -> the CPU oracle on a bounded token sample (rank 0, N = 1)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

# P:345 sets CUDA_DEVICE_MAX_CONNECTIONS=1 so that, in ONE hardware work queue, a
# communication kernel enqueued before the next GEMM is launched first.  This
# library's schedule instead gives the communication stream its own queue (high
# priority, gated by device-side chunk counters); with a single queue the dW
# GEMM queued behind the dX GEMM would block the chunk all-reduces
# (head-of-line), so the default connection count is kept.
# An explicit setting in the environment is respected.

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TFLOP/s/GPU and exposed-comm ms per GPT layer fwd+bwd at 1/2/4/8 B200 per mesh"
VALUE_SCOPE = "whole job: linear-block FLOPs of all N GPUs / step time (per GPU: tflops_per_gpu)"


def default_shape(world: int) -> tuple[int, int, str]:
    """(hidden, heads, BASELINE config) bench.py runs at N GPUs by default."""
    if world == 1:
        return 12288, 96, "cfg 5 shape (largest single-GPU configuration)"
    if world == 8:
        return 5120, 40, "cfg 4 (north_star target)"
    return 4096, 32, "cfg 2"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="atp", choices=["atp", "reference"])
    p.add_argument("--hidden", type=int, default=0, help="0 = the per-N default (see the module docstring)")
    p.add_argument("--heads", type=int, default=0)
    p.add_argument("--ffn", type=int, default=0, help="default 4*hidden")
    p.add_argument("--batch", type=int, default=4)
    p.add_argument("--seq", type=int, default=2048)
    p.add_argument("--layers", type=int, default=0,
                   help="linear block: stack of L layers as one pipeline (atp_layer_stack_fwd_bwd; SURVEY §8(d) "
                        "L_bench) -- 0 = 4 at N>1 (a layer's last all-reduce overlaps the next layer's GEMM), "
                        "1 at N=1 (no communication to overlap)")
    p.add_argument("--layer", default="linear", choices=["linear", "gpt"],
                   help="linear: the north_star linear block (default); gpt: the full pre-LN layer "
                        "(LayerNorm + causal softmax attention core, SURVEY NEXT #1)")
    p.add_argument("--mesh", default="", help="d1xd2; default: atp_search on the probed HCM + calibration")
    p.add_argument("--no-probe", action="store_true",
                   help="N>1: skip atp_probe_hcm; search on the uniform 900 GB/s NVSwitch HCM, plan at --busbw")
    p.add_argument("--probe-mib", type=int, default=256, help="largest probe message (MiB); 64 MiB and the "
                   "layer's chunk size are also measured")
    p.add_argument("--p2p-disable", action="store_true",
                   help="N>1 topology stress (P:373, the paper's IC1): NCCL_P2P_DISABLE=1 before NCCL init, "
                        "then probe -> calibrated search as usual")
    p.add_argument("--fused-ar", action="store_true",
                   help="N>1: fused peer-memory all-reduce (CUDA IPC) instead of NCCL on the data path")
    p.add_argument("--nccl-only", action="store_true",
                   help="N>1 linear block: no variant selection (plain NCCL step)")
    p.add_argument("--try-fused", action="store_true",
                   help="N>1 linear block: also time the fused GEMM->reduce-scatter->all-gather path against NCCL "
                        "and run the faster (with --try-gated: also both chunk-gated)")
    p.add_argument("--try-gated", action="store_true",
                   help="N>1 linear block: also time NCCL with chunk gating and run the faster")
    p.add_argument("--gated", action="store_true",
                   help="N>1: chunk-gated GEMMs (the next stage's GEMM waits per chunk for the all-reduce tail)")
    p.add_argument("--no-baseline", action="store_true", help="N>1: skip the DeviceMesh(N,1) c=1 baseline")
    p.add_argument("--chunks", type=int, default=0,
                   help="0 = 1 at N=1; at N>1 chosen by atp_plan_chunks from measured compute + probed busBW")
    p.add_argument("--busbw", type=float, default=725.0,
                   help="all-reduce bus GB/s for the chunk planner when the probe does not run")
    p.add_argument("--gemm-ctas", type=int, default=-1, help="GEMM CTA cap (default: all SMs at N=1, SMs-16 else)")
    p.add_argument("--share-gpu", action="store_true",
                   help="TEST ONLY: N>1 ranks share cuda:0 (distinct NCCL_HOSTID per rank, NCCL over sockets); "
                        "exercises the multi-process data path on a 1-GPU box, timings meaningless")
    p.add_argument("--no-graph", action="store_true",
                   help="time direct calls instead of the step captured as one CUDA graph (atp_graph_*)")
    p.add_argument("--seed", type=int, default=2301)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-cupti", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU-oracle sample duration")
    p.add_argument("--peaks", default=os.path.join(ROOT, "MEASURED_PEAKS.json"))
    a = p.parse_args()
    return a


# ----------------------------------------------------------------------------- helpers
def layer_flops(T: int, h: int, F: int) -> float:
    """Linear-block FLOPs of one layer fwd+bwd: fwd 2T(3h^2 + h^2 + 2hF), bwd 2x (= 72Th^2 at F=4h)."""
    return 3.0 * 2.0 * T * (3 * h * h + h * h + 2 * h * F)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms during a region."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.lines = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={device_index}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.5)
        except (OSError, ValueError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def stop(self, t0: float, t1: float) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, pw, reasons, n = [], [], [], set(), 0
        for (tw, line) in self.lines:
            if not (t0 - 0.15 <= tw <= t1 + 0.15):
                continue
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
                pw.append(float(parts[3]))
            except ValueError:
                continue
            n += 1
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": n, "power_w_max": max(pw) if pw else None}


def peaks(path: str) -> dict:
    try:
        with open(path) as f:
            p = json.load(f)
        return {"bf16_tflops": p["bf16_tflops"], "bf16_tflops_sustained": p.get("bf16_tflops_sustained"),
                "hbm_gbs": p["hbm_gbs"], "source": "measured (MEASURED_PEAKS.json)"}
    except (OSError, KeyError, ValueError):
        # /opt/skills/guides/B200_PROFILING.md fallback
        return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0,
                "source": "fallback (B200_PROFILING.md)"}


def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        return max((i.get("num_threads", 1) for i in threadpool_info()), default=os.cpu_count())
    except Exception:  # noqa: BLE001
        return os.cpu_count()


def oracle_weights(h: int, F: int, seed: int) -> dict:
    """The layer's global weights and biases in float64 (generated once, not timed)."""
    import numpy as np
    import datagen

    shapes = datagen.layer_shapes(8, h, F)
    return {k: datagen.tensor(k, s, seed=seed).astype(np.float64) for k, s in shapes.items() if k not in ("x", "dz")}


def cpu_oracle_run(w: dict, T_s: int, h: int, heads: int, seed: int) -> float:
    """Time the CPU oracle (fp64 NumPy SPMD simulation at mesh (1,1)) on T_s tokens."""
    import numpy as np
    import datagen
    from oracle import layer as olayer

    g = dict(w, x=datagen.tensor("x", (T_s, h), seed=seed).astype(np.float64),
             dz=datagen.tensor("dz", (T_s, h), seed=seed).astype(np.float64))
    t0 = time.perf_counter()
    olayer.run_layer(g, 1, 1, heads, 1)
    return time.perf_counter() - t0


def sample_tokens(w, h, heads, seed, target_s: float) -> tuple[int, float, float]:
    """Token count whose oracle run takes ~target_s (the time is affine in the
    tokens: fixed weight copies + per-token GEMMs); two calibration points."""
    t_a = cpu_oracle_run(w, 16, h, heads, seed)
    t_b = cpu_oracle_run(w, 208, h, heads, seed)  # a mid-size point: the per-token cost grows with T
    per_tok = max((t_b - t_a) / 192.0, 1e-6)
    fixed = max(t_a - 16 * per_tok, 0.0)
    T_s = int(max(16, min(8192, (target_s - fixed) / per_tok)) // 8 * 8)
    return T_s, fixed, per_tok


def cpu_baseline(h: int, F: int, heads: int, seed: int, target_s: float) -> dict:
    w = oracle_weights(h, F, seed)
    T_s, _, _ = sample_tokens(w, h, heads, seed, target_s)
    t = cpu_oracle_run(w, T_s, h, heads, seed)
    fl = layer_flops(T_s, h, F)
    return {"value": fl / t / 1e12, "unit": "TFLOP/s", "cores": blas_threads(), "kind": "oracle",
            "sample": f"{T_s} of 8192 tokens of the same layer (h={h}, F={F}), fp64 NumPy SPMD simulation at "
                      f"DeviceMesh(1,1) incl. its per-call weight shard copies, {t:.1f} s",
            "seconds": t, "tokens": T_s}


def traffic_for(h: int, T: int):
    """Measured DRAM bytes (read + write) per GEMM launch of this workload's step,
    from the committed ncu --set full capture (profiles/*_gemm_traffic.json,
    written by scripts/ncu_traffic.py); None when there is none for (h, T)."""
    import glob

    best = None
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_gemm_traffic.json"))):
        try:
            d = json.load(open(f))
        except Exception:  # noqa: BLE001
            continue
        if d.get("hidden") == h and d.get("tokens") == T and d.get("gemm_launches"):
            best = {"dram_bytes_per_gemm_launch": d["gemm_dram_bytes"] / d["gemm_launches"],
                    "algorithmic_bytes_per_gemm_launch": d.get("gemm_algorithmic_bytes", 0) / d["gemm_launches"],
                    "source": os.path.relpath(f, ROOT)}
    return best


def gpt_flops(T: int, h: int, F: int, seq: int) -> float:
    """FLOPs the full causal layer performs fwd+bwd: the linear block plus the
    attention core (forward 4*d per visible (query, key) pair and head = 2(s+1)Th
    for causal rows; backward 2.5x)."""
    return layer_flops(T, h, F) + 7.0 * (seq + 1) * T * h


def gpt_flops_paper(T: int, h: int, seq: int) -> float:
    """The paper's per-layer count 72bsh^2 + 12bs^2h (non-causal core, F = 4h)."""
    return 72.0 * T * h * h + 12.0 * T * seq * h


def cpu_baseline_gpt(h: int, F: int, heads: int, seq: int, seed: int) -> dict:
    """The full-layer oracle (fp64 NumPy, oracle/gpt.py) on one whole sequence."""
    import datagen
    from oracle import gpt

    g = {k: v.astype("float64") for k, v in datagen.gpt_globals(seq, h, F, seed).items()}
    t0 = time.time()
    fw = gpt.dense_forward(g, heads, seq)
    gpt.dense_backward(g, fw, g["dz"], heads, seq)
    t = time.time() - t0
    return {"value": gpt_flops(seq, h, F, seq) / t / 1e12, "unit": "TFLOP/s", "cores": blas_threads(),
            "kind": "oracle", "sample": f"1 sequence ({seq} tokens) of the full layer (h={h}, F={F}, {heads} heads, "
                                        f"causal), fp64 NumPy dense oracle, {t:.1f} s", "seconds": t, "tokens": seq}


def _quiet(fn):
    """Run fn with fd 1 redirected to stderr (NCCL prints its version banner on
    stdout at communicator init; stdout carries only the JSON line)."""
    sys.stdout.flush()
    saved_fd = os.dup(1)
    os.dup2(2, 1)
    try:
        return fn()
    finally:
        sys.stdout.flush()
        os.dup2(saved_fd, 1)
        os.close(saved_fd)


def note(msg: str) -> None:
    """Progress marker on stderr (rank-prefixed by the caller): localises a hang."""
    print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def emit(obj: dict) -> None:
    print(json.dumps(obj), flush=True)


def union_ms(iv) -> float:
    """Length (ms) of the union of [start_ns, end_ns) intervals."""
    tot, cur_s, cur_e = 0, None, None
    for s, e in sorted(iv):
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                tot += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    if cur_e is not None:
        tot += cur_e - cur_s
    return tot / 1e6


def cupti_kernels(run, stream, n: int):
    """Kernel records (name, start_ns, end_ns) of n launches of `run` (the
    graph-launched step) from a CUPTI activity trace (torch.profiler/kineto).
    Every record is a kernel of the step as it executes inside the graph."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(n):
            run(stream)
        torch.cuda.synchronize()
    out = []
    for e in prof.profiler.kineto_results.events():
        if e.device_type() != torch.autograd.DeviceType.CUDA:
            continue
        nm = e.name()
        if nm.startswith("Memcpy") or nm.startswith("Memset") or "cudaStream" in nm:
            continue
        out.append((nm, e.start_ns(), e.end_ns()))
    return out


def kernel_class(name: str) -> str:
    if "gemm_sm100" in name or "gemm_f32" in name:
        return "gemm"
    if "attn" in name:
        return "attention"
    if "nccl" in name.lower():
        return "nccl"
    return "elementwise"


# ----------------------------------------------------------------------------- reference arm
def run_reference(a) -> None:
    """The CPU oracle, as it stands, timed on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    dh, dheads, cfg = default_shape(world)
    h = a.hidden or dh
    heads = a.heads or dheads
    F = a.ffn or 4 * h
    w = oracle_weights(h, F, a.seed)
    # one bounded sample per step, sized so the whole run stays within a few minutes
    budget = 150.0 / max(1, a.steps + a.warmup)
    T_s, fixed, per_tok = sample_tokens(w, h, heads, a.seed, budget)
    for _ in range(a.warmup):
        cpu_oracle_run(w, T_s, h, heads, a.seed)
    times = [cpu_oracle_run(w, T_s, h, heads, a.seed) for _ in range(a.steps)]
    t = sum(times) / len(times)
    v = layer_flops(T_s, h, F) / t / 1e12
    threads = blas_threads()
    emit({"impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": a.gpus, "steps": a.steps,
          "warmup": a.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
          "vs_baseline": None, "dtype": "f64", "data": "synthetic",
          "config": {"workload": f"gpt-layer linear block h{h} a{heads} ffn{F} ({cfg}), {T_s}-token sample per step "
                                 f"(of b{a.batch} s{a.seq})", "mesh": [1, 1], "tokens_per_step": T_s,
                     "hidden": h, "heads": heads, "ffn": F},
          "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
                           "sample": f"{T_s} tokens per step, fp64 NumPy SPMD simulation at DeviceMesh(1,1) "
                                     f"(fixed per-call cost ~{fixed:.1f} s: weight shard copies)"},
          "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
          "gpu_launches": 0})


# ----------------------------------------------------------------------------- ATP arm
def main() -> None:
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    if a.p2p_disable:
        os.environ["NCCL_P2P_DISABLE"] = "1"  # read by NCCL at communicator init (IC1)
    if a.share_gpu:
        os.environ["NCCL_HOSTID"] = f"atp-shared-gpu-rank{rank}"  # NCCL rejects two ranks on one device of one host
        os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
        local_rank = 0

    import torch
    import torch.distributed as dist

    import paper_2301_08658_b200 as atp
    from paper_2301_08658_b200 import _abi

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        _quiet(lambda: dist.init_process_group("nccl", device_id=dev))  # eager NCCL init prints its banner

    dh, dheads, cfg_name = default_shape(world)
    h = a.hidden or dh
    heads = a.heads or dheads
    if a.hidden and not a.heads:
        heads = max(1, h // 128)
    F = a.ffn or 4 * h
    T = a.batch * a.seq
    gpt_mode = a.layer == "gpt"
    L = 1 if gpt_mode else (a.layers or (4 if world > 1 else 1))

    def new_uid() -> bytes:
        uid = atp.atp_get_unique_id() if rank == 0 else bytes(128)
        if world > 1:
            obj = [uid]
            dist.broadcast_object_list(obj, src=0)
            uid = obj[0]
        return uid

    # ---- mesh: explicit, or ATP's search (§3.5) on the HCM measured by
    # atp_probe_hcm (S1) with the per-mesh calibration, or with
    # --no-probe on the single-layer NVSwitch HCM (P:488, 900 GB/s per direction).
    plan = plan_hcm = None
    probe = None
    mesh_source = "flag" if a.mesh else ("N=1" if world == 1 else "")
    busbw, busbw_source = a.busbw, "--busbw"
    if world > 1 and not a.mesh:
        layers, calib = [atp.HcmLayer(world, 900.0, 900.0)], None
        mesh_source = "atp_search(uniform 900 GB/s HCM)"
        if not a.no_probe:
            try:
                pm = _quiet(lambda: atp.Mesh.distributed(world, 1, rank, new_uid(), local_rank))
                chunk_bytes = 2 * (T // 4) * (4 * h // max(1, world // 2))
                big = a.probe_mib << 20
                sizes = tuple(sorted({min(64 << 20, big), big, chunk_bytes}))
                scratch = torch.empty(max(big, chunk_bytes) + 64, dtype=torch.uint8, device=dev)
                t0 = time.time()
                layers, matrix, calib = atp.atp_probe_hcm(pm, scratch, msg_bytes=sizes, calib_bytes=chunk_bytes,
                                                          iters=10)
                pm.destroy()
                del scratch
                probe = {"hcm": [vars(l) for l in layers], "p2p_matrix_gbps": matrix,
                         "calibration_algbw_gbps": {f"{d1}x{d2}": v for (d1, d2), v in calib.items()},
                         "msg_bytes": list(sizes), "calib_bytes": chunk_bytes, "seconds": time.time() - t0,
                         "nccl_p2p_disable": bool(a.p2p_disable)}
                busbw, busbw_source = layers[0].group_gbps, f"probe: {world}-rank all-reduce busBW (GroupBW)"
                mesh_source = "atp_search(probed HCM + calibration, P:482)"
            except Exception as e:  # noqa: BLE001
                print(f"probe failed, using the uniform HCM: {e}", file=sys.stderr)
                probe = {"error": str(e)}
        plan_hcm = atp.atp_search(layers, 1, a.batch, a.seq, h, heads, 2)
        plan = atp.atp_search(layers, 1, a.batch, a.seq, h, heads, 2, calibration=calib) if calib else plan_hcm
        d1, d2 = plan["chosen"]
        if calib:
            # bus bandwidth of the chosen mesh's own groups (B'_k = B_k 2(d_k-1)/d_k): the planner's comm rate
            b1, b2 = calib.get((d1, d2), (None, None))
            bus = [b * 2.0 * (d - 1) / d for b, d in ((b1, d1), (b2, d2)) if b and d > 1]
            if bus:
                busbw, busbw_source = min(bus), f"probe: calibrated busBW of DeviceMesh({d1},{d2})'s groups"
    elif a.mesh:
        d1, d2 = (int(v) for v in a.mesh.lower().split("x"))
    else:
        d1, d2 = 1, 1
    assert d1 * d2 == world

    note(f"rank {rank}: mesh {d1}x{d2} ({mesh_source})")
    ctas = a.gemm_ctas if a.gemm_ctas >= 0 else (0 if world == 1 else 132)
    stream = torch.cuda.Stream(device=dev)  # a capturable (non-legacy) stream for every launch of the bench
    torch.cuda.set_stream(stream)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def maxrank(ms: float) -> float:
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    def timed(n_steps: int, fn) -> float:
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(n_steps):
            fn(stream)
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / n_steps
        barrier()
        return maxrank(ms)

    def make_mesh(m1, m2):
        m = _quiet(lambda: atp.Mesh.distributed(m1, m2, rank, new_uid(), local_rank))
        m.set_gemm_ctas(ctas)
        return m

    mesh = make_mesh(d1, d2)
    mesh.set_gating(a.gated)
    if a.fused_ar and world > 1:
        mesh.enable_fused_ar(T * max(3 * h // d1, F // d1, h // d2) * 2)  # one stage's partials [T, widest], bf16

    def alloc(m1, m2, n_layers=None):
        n_layers = L if n_layers is None else n_layers
        if gpt_mode:
            return atp.alloc_gpt_rank(m1, m2, rank, T, h, F, heads, dev, a.seed)
        if n_layers > 1:  # list of per-layer buffer dicts, chained (layer l+1's x is layer l's z)
            return atp.alloc_layer_stack(m1, m2, rank, T, h, F, dev, a.seed, n_layers)
        return atp.alloc_layer_rank(m1, m2, rank, T, h, F, dev, a.seed)

    def make_call(m, bb, c):
        if gpt_mode:
            return atp.GptCall(m, [bb], T, h, F, heads, a.seq, c, True)
        if isinstance(bb, list):
            return atp.LayerStackCall(m, [[b] for b in bb], T, h, F, heads, c)
        return atp.LayerCall(m, [bb], T, h, F, heads, c, True)

    first = lambda bb: bb[0] if isinstance(bb, list) else bb  # the stack's input layer
    last = lambda bb: bb[-1] if isinstance(bb, list) else bb  # ... and output layer

    bufs = alloc(d1, d2)

    # ---- chunk count (N>1, --chunks 0): the compute side of each candidate is
    # measured with the all-reduces disabled, then atp_plan_chunks (the overlap
    # model of §4.1/§4.2 inside libatp) predicts each step at the probed bus
    # bandwidth and picks the fastest (same on every rank: max over ranks first).
    chunk_choice = None
    if a.chunks:
        chunks = a.chunks
    elif world == 1 or (d1 == 1 and d2 == 1):
        chunks = 1
    elif gpt_mode:
        chunks = min(2, a.batch)  # whole sequences; "2 or 4" (2: attention occupancy)
    else:
        comp = {}
        _abi.check(_abi.lib().atp_mesh_set_comm_enabled(mesh.handle, 0))
        for c in (1, 2, 4, 8):
            if T % c or (T // c) % 8:
                continue
            cc = make_call(mesh, bufs, c)
            for _ in range(2):
                cc(stream)
            comp[c] = timed(5, cc)
        _abi.check(_abi.lib().atp_mesh_set_comm_enabled(mesh.handle, 1))
        chunks, pred = atp.atp_plan_chunks(T, h, F, d1, d2, comp, busbw)
        chunk_choice = {"compute_ms": comp, "predicted_ms": {c: v[0] for c, v in pred.items()},
                        "predicted_exposed_ms": {c: v[1] for c, v in pred.items()}, "busbw_gbs": busbw,
                        "busbw_source": busbw_source, "chosen": chunks, "planner": "libatp atp_plan_chunks"}
    call = make_call(mesh, bufs, chunks)
    note(f"rank {rank}: chunks {chunks}, layers {L}; warm-up")

    for _ in range(max(3, a.warmup)):
        call(stream)
    torch.cuda.synchronize()

    # ---- the step as one CUDA graph (atp_graph_*): host cost per step = one
    # cudaGraphLaunch; direct calls stay in use for the comm-disabled twin and
    # the event-profiled pass (per-launch events cannot be captured)
    graphs, capture_errors = [], []

    def as_graph(m, c):
        if a.no_graph:
            return c
        try:
            g = atp.Graph.capture(m, c, stream)
        except Exception as e:  # noqa: BLE001  (fused peer-memory meshes refuse capture)
            capture_errors.append(str(e))
            return c
        graphs.append(g)
        return g

    run = as_graph(mesh, call)
    graph_note = ("direct calls (--no-graph)" if a.no_graph else
                  f"direct calls (graph capture unavailable: {capture_errors[0]})" if capture_errors else
                  "step captured once as a CUDA graph, one cudaGraphLaunch per step")
    for _ in range(2):
        run(stream)
    torch.cuda.synchronize()

    # ---- N>1 linear block: NCCL all-reduce (graph-captured step) vs chunk gating
    # and the fused peer-memory all-reduce, timed on this box; the faster one runs
    # the measured steps.  Timings are max-reduced over ranks: every rank agrees.
    ar_choice = None
    meshes = [mesh]
    if world > 1 and not gpt_mode and not a.fused_ar and not a.nccl_only and not a.gated and \
            (a.try_gated or a.try_fused):
        times, runners = {}, {}
        try:
            note(f"rank {rank}: variant nccl")
            times["nccl"], runners["nccl"] = timed(10, run), (mesh, call, run, False, graph_note)
            if a.try_gated:
                note(f"rank {rank}: variant nccl+gated")
                mesh.set_gating(True)
                run_g = as_graph(mesh, call)
                for _ in range(2):
                    run_g(stream)
                times["nccl+gated"] = timed(10, run_g)
                runners["nccl+gated"] = (mesh, call, run_g, True, graph_note)
                mesh.set_gating(False)
            if a.try_fused:
                mesh_f = make_mesh(d1, d2)
                meshes.append(mesh_f)
                mesh_f.enable_fused_ar(T * max(3 * h // d1, F // d1, h // d2) * 2)
                call_f = make_call(mesh_f, bufs, chunks)
                note_f = "direct calls (fused peer-memory mesh keeps cross-rank state: no graph capture)"
                for gated in ((False, True) if a.try_gated else (False,)):
                    note(f"rank {rank}: variant fused gated={gated}")
                    mesh_f.set_gating(gated)
                    for _ in range(3):
                        call_f(stream)
                    key = "fused+gated" if gated else "fused"
                    times[key] = timed(10, call_f)
                    runners[key] = (mesh_f, call_f, call_f, gated, note_f)
        except Exception as e:  # noqa: BLE001  (keeps the NCCL step)
            ar_choice = {"error": str(e)}
            mesh.set_gating(False)
        if times:
            best = min(times, key=times.get)
            ar_choice = dict(ar_choice or {}, timed_ms=times, chosen=best)
            mesh, call, run, chosen_gating, graph_note = runners[best]
            mesh.set_gating(chosen_gating)
            a.gated = chosen_gating

    # ---- timed region (clocks sampled during it)
    note(f"rank {rank}: timed region")
    sampler = ClockSampler(local_rank)
    import ctypes as C

    n0 = C.c_uint64()
    _abi.check(_abi.lib().atp_launch_count(C.byref(n0)))
    t0 = time.time()
    ms = timed(a.steps, run)
    t1 = time.time()
    n1 = C.c_uint64()
    _abi.check(_abi.lib().atp_launch_count(C.byref(n1)))
    clocks = sampler.stop(t0, t1)
    launches = int(n1.value - n0.value)

    fl = gpt_flops(T, h, F, a.seq) if gpt_mode else L * layer_flops(T, h, F)
    gemm_fl = L * layer_flops(T, h, F) / world  # the GEMM FLOPs of one rank per step
    value = fl / (ms * 1e-3) / 1e12
    per_gpu = value / world

    # ---- comm-disabled twin (exposed communication)
    exposed = 0.0
    ms_nocomm = ms
    if d1 > 1 or d2 > 1:
        _abi.check(_abi.lib().atp_mesh_set_comm_enabled(mesh.handle, 0))
        ms_nocomm = timed(max(10, a.steps // 2), call)
        _abi.check(_abi.lib().atp_mesh_set_comm_enabled(mesh.handle, 1))
        exposed = max(0.0, ms - ms_nocomm)

    # ---- roofline of the dominant kernel (the tcgen05 GEMM): GEMM time and its
    # share of the step from a CUPTI trace of the SAME graph-launched step
    pk = peaks(a.peaks)
    timed_s = ms * a.steps / 1e3
    throttled = bool(clocks.get("sm_mhz") and clocks.get("sm_max_mhz") and
                     clocks["sm_mhz"] < 0.9 * clocks["sm_max_mhz"] and "sw_power_cap" in clocks.get("reasons", []))
    use_sustained = throttled and timed_s >= 2.0 and pk["bf16_tflops_sustained"]
    peak_tc = pk["bf16_tflops_sustained"] if use_sustained else pk["bf16_tflops"]
    peak_rule = ("sustained: this run's timed region lasted %.1f s with SM clocks at %s of %s MHz under sw_power_cap"
                 % (timed_s, clocks.get("sm_mhz"), clocks.get("sm_max_mhz")) if use_sustained else
                 "burst: the timed region was not a seconds-long power-capped run (%.2f s, median %s of %s MHz)"
                 % (timed_s, clocks.get("sm_mhz"), clocks.get("sm_max_mhz")))
    n_prof = max(3, min(a.steps, 10))
    roofline = {"bound": "tensor", "unit": "TFLOP/s", "peak": peak_tc, "peak_rule": peak_rule,
                "peak_burst": pk["bf16_tflops"], "peak_sustained": pk["bf16_tflops_sustained"],
                "peak_source": pk["source"], "kernel": "gemm_sm100_kernel (tcgen05; all GEMM launches of the step)",
                "traffic": None}
    cupti = None
    if not a.no_cupti:
        try:
            ks = cupti_kernels(run, stream, n_prof)
            by = {}
            for nm, s, e in ks:
                by.setdefault(kernel_class(nm), []).append((s, e))
            span = (max(e for _, _, e in ks) - min(s for _, s, _ in ks)) / 1e6 / n_prof if ks else None
            gemm_ms = union_ms(by.get("gemm", [])) / n_prof
            cupti = {"kernels_per_step": len(ks) / n_prof,
                     "gemm_launches_per_step": len(by.get("gemm", [])) / n_prof,
                     "ms_per_step_by_class": {k: union_ms(v) / n_prof for k, v in by.items()},
                     "traced_step_span_ms": span, "steps_traced": n_prof,
                     "source": "CUPTI activity trace (torch.profiler/kineto) of the graph-launched step, "
                               "kernel intervals merged per class (PDL overlap counted once)"}
            if gemm_ms > 0:
                roofline["achieved"] = gemm_fl / (gemm_ms * 1e-3) / 1e12
                roofline["frac"] = roofline["achieved"] / peak_tc
                roofline["frac_burst"] = roofline["achieved"] / pk["bf16_tflops"]
                if pk["bf16_tflops_sustained"]:
                    roofline["frac_sustained"] = roofline["achieved"] / pk["bf16_tflops_sustained"]
                roofline["gemm_ms_per_step"] = gemm_ms
                roofline["gemm_share_of_step"] = gemm_ms / ms
                roofline["avg_gemm_launch_ms"] = gemm_ms / max(1e-9, cupti["gemm_launches_per_step"])
        except Exception as e:  # noqa: BLE001
            cupti = {"error": f"{type(e).__name__}: {e}"}
    # cross-check: per-launch CUDA events recorded by the executor on the launching streams (direct calls)
    prof = _abi.Profile()
    n_ev = max(5, min(a.steps, 20))
    _abi.check(_abi.lib().atp_profile_begin(mesh.handle))
    ms_prof = timed(n_ev, call)
    _abi.check(_abi.lib().atp_profile_end(mesh.handle, C.byref(prof)))
    ev_gemm_ms = prof.ms[0] / n_ev
    event_profile = {"gemm_ms_per_step": ev_gemm_ms,
                     "gemm_tflops": (prof.flops[0] / n_ev) / (ev_gemm_ms * 1e-3) / 1e12 if ev_gemm_ms > 0 else None,
                     "gemm_launches_per_step": prof.launches[0] / n_ev,
                     "elementwise_ms_per_step": prof.ms[1] / n_ev,
                     "elementwise_gbs": (prof.bytes[1] / max(prof.ms[1], 1e-9)) / 1e6,
                     "allreduce_ms_per_step": prof.ms[2] / n_ev,
                     "allreduce_busbw_gbs": (prof.bytes[2] / max(prof.ms[2], 1e-9)) / 1e6 if prof.ms[2] > 0 else None,
                     "profiled_ms_per_step": ms_prof,
                     "note": "direct calls with a CUDA event pair around every launch (no graph, no PDL)"}
    if "achieved" not in roofline and ev_gemm_ms > 0:  # CUPTI unavailable: fall back to the events
        roofline["achieved"] = event_profile["gemm_tflops"]
        roofline["frac"] = roofline["achieved"] / peak_tc
        roofline["gemm_share_of_step"] = ev_gemm_ms / ms_prof
    tr = traffic_for(h, T) if world == 1 else None
    if tr:
        roofline["traffic"] = tr["dram_bytes_per_gemm_launch"]
        roofline["traffic_detail"] = tr
    roofline["layer_roofline_frac"] = (fl / world / (peak_tc * 1e12)) / (ms * 1e-3)
    if gpt_mode:
        att_ms = prof.ms[3] / n_ev
        roofline.update({
            "attention_ms_per_step": att_ms,
            "attention_tflops": (prof.flops[3] / n_ev) / (att_ms * 1e-3) / 1e12 if att_ms > 0 else None,
            "attention_share_of_step": att_ms / ms_prof if ms_prof > 0 else None})

    # ---- the stack against one layer per call ("Headline =
    # steady-state per layer; L=1 is also reported")
    single = None
    if L > 1:
        try:
            b1 = alloc(d1, d2, 1)
            c1 = make_call(mesh, b1, chunks)
            for _ in range(3):
                c1(stream)
            ms1 = timed(max(5, a.steps // 2), as_graph(mesh, c1))
            single = {"ms_per_step": ms1, "ms_per_layer_in_stack": ms / L, "stack_gain": ms1 / (ms / L)}
            del b1
        except Exception as e:  # noqa: BLE001
            single = {"error": str(e)}

    # ---- Megatron-style baseline (north_star): the same library on DeviceMesh(N,1), 1 chunk
    note(f"rank {rank}: extra passes (baseline / e2e)")
    baseline = None
    if world > 1 and not a.no_baseline and not gpt_mode and ((d1, d2) != (world, 1) or chunks != 1):
        try:
            mb = make_mesh(world, 1)
            meshes.append(mb)
            bb = alloc(world, 1)
            cb = make_call(mb, bb, 1)
            for _ in range(3):
                cb(stream)
            rb = as_graph(mb, cb)
            ms_b = timed(a.steps, rb)
            _abi.check(_abi.lib().atp_mesh_set_comm_enabled(mb.handle, 0))
            ms_b0 = timed(max(10, a.steps // 2), cb)
            _abi.check(_abi.lib().atp_mesh_set_comm_enabled(mb.handle, 1))
            baseline = {"mesh": [world, 1], "chunks": 1, "layers": L, "ms_per_step": ms_b,
                        "tflops_per_gpu": fl / (ms_b * 1e-3) / 1e12 / world,
                        "exposed_comm_ms": max(0.0, ms_b - ms_b0), "ms_per_step_comm_disabled": ms_b0,
                        "speedup_of_atp_step": ms_b / ms}
            del bb
        except Exception as e:  # noqa: BLE001
            baseline = {"error": str(e)}

    # ---- e2e: every step's inputs (X, dZ) H2D from pinned host memory and its
    # result (the bias gradients) D2H, through the public API.  Inputs are
    # double-buffered: step i+1's copy runs on a copy stream while step i computes.
    e2e = None
    if not a.no_e2e:
        hx = first(bufs)["x"].cpu().pin_memory()
        hdz = last(bufs)["dz"].cpu().pin_memory()
        res = [first(bufs)[k] for k in ("dbqkv", "dbo", "db1", "db2")]
        hres = [torch.empty(r.shape, dtype=r.dtype).pin_memory() for r in res]
        h2d = hx.numel() * hx.element_size() + hdz.numel() * hdz.element_size()
        d2h = sum(r.numel() * r.element_size() for r in res)
        if isinstance(bufs, list):  # second input set: own x (layer 0) and dz (last layer), the rest shared
            bufs_b = [dict(b) for b in bufs]
            bufs_b[0]["x"] = torch.empty_like(bufs[0]["x"])
            bufs_b[-1]["dz"] = torch.empty_like(bufs[-1]["dz"])
        else:
            bufs_b = dict(bufs, x=torch.empty_like(bufs["x"]), dz=torch.empty_like(bufs["dz"]))
        sets = [(bufs, run), (bufs_b, as_graph(mesh, make_call(mesh, bufs_b, chunks)) if run is not call else
                                  make_call(mesh, bufs_b, chunks))]
        copy_stream = torch.cuda.Stream()
        copied = [torch.cuda.Event(), torch.cuda.Event()]
        done = [torch.cuda.Event(), torch.cuda.Event()]

        def run_e2e(n):
            with torch.cuda.stream(copy_stream):
                first(sets[0][0])["x"].copy_(hx, non_blocking=True)
                last(sets[0][0])["dz"].copy_(hdz, non_blocking=True)
                copied[0].record(copy_stream)
            for i in range(n):
                cur, nxt = i % 2, (i + 1) % 2
                stream.wait_event(copied[cur])
                sets[cur][1](stream)
                done[cur].record(stream)
                for r, hr in zip(res, hres):
                    hr.copy_(r, non_blocking=True)
                if i + 1 < n:
                    with torch.cuda.stream(copy_stream):
                        if i >= 1:
                            copy_stream.wait_event(done[nxt])
                        first(sets[nxt][0])["x"].copy_(hx, non_blocking=True)
                        last(sets[nxt][0])["dz"].copy_(hdz, non_blocking=True)
                        copied[nxt].record(copy_stream)

        run_e2e(3)
        barrier()
        n_e2e = max(5, min(a.steps, 30))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        copy_stream.wait_event(e0)
        run_e2e(n_e2e)
        e1.record(stream)
        e1.synchronize()
        ms_e2e = maxrank(e0.elapsed_time(e1) / n_e2e)
        e2e = {"value": fl / (ms_e2e * 1e-3) / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d * world,
               "d2h_bytes_per_step": d2h * world, "ms_per_step": ms_e2e,
               "api": ("paper_2301_08658_b200.GptCall -> atp_gpt_layer_fwd_bwd (C ABI)" if gpt_mode else
                       "paper_2301_08658_b200.LayerCall -> atp_layer_fwd_bwd (C ABI)"),
               "note": "every rank copies its X, dZ shards H2D every step (double-buffered on a copy stream) and "
                       "reads its bias gradients D2H; bytes summed over ranks"}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = (cpu_baseline_gpt(h, F, heads, a.seq, a.seed) if gpt_mode
               else cpu_baseline(h, F, heads, a.seed, a.cpu_seconds))

    for g in graphs:
        g.destroy()
    for m in meshes:
        m.destroy()
    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "value_scope": VALUE_SCOPE, "n_gpus": world,
            "steps": a.steps, "warmup": max(3, a.warmup), "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": (f"full pre-LN GPT layer (LN + QKV + causal softmax attention + Out + LN + MLP, "
                                    f"fwd+bwd) h{h} a{heads} ffn{F} s{a.seq} b{a.batch}, DeviceMesh({d1},{d2}), "
                                    f"chunks {chunks}") if gpt_mode else
                                   (f"gpt-layer linear block (QKV/Out/FC1/FC2 fwd+bwd) h{h} a{heads} ffn{F} "
                                    f"s{a.seq} b{a.batch} ({cfg_name}), DeviceMesh({d1},{d2}), chunks {chunks}"
                                    + (f", stack of {L} layers as one pipeline (value counts all {L})" if L > 1
                                       else "")),
                       "mesh": [d1, d2], "chunks": chunks, "layers": L, "tokens": T, "hidden": h, "heads": heads,
                       "ffn": F, "nccl_max_ctas": int(os.environ.get("ATP_NCCL_MAX_CTAS", "16")),
                       "parallelism": f"atp{d1}x{d2}", "gemm_ctas": ctas,
                       "allreduce": ("fused peer-memory kernel" if ((a.fused_ar or str((ar_choice or {}).get("chosen", "")).startswith("fused"))
                                                                    and world > 1) else "nccl"),
                       "gated": bool(a.gated and world > 1), "mesh_source": mesh_source, "launch": graph_note,
                       "nccl_p2p_disable": bool(a.p2p_disable),
                       **({"shared_gpu": "TEST ONLY: all ranks on cuda:0, NCCL over sockets; timings meaningless"}
                          if a.share_gpu else {}),
                       "l2": "working set > 126 MB L2 (weights+activations, GBs), no flush"},
            "tflops_per_gpu": per_gpu, "exposed_comm_ms": exposed, "ms_per_step_comm_disabled": ms_nocomm,
            "exposed_comm_frac": exposed / ms if ms > 0 else None,
            "flops_per_step": fl, "clocks": clocks, "gpu_launches": launches,
            "roofline": roofline, "e2e": e2e, "cpu_baseline": cpu,
            "kernel_trace": cupti, "event_profile": event_profile,
        }
        if chunk_choice is not None:
            out["chunk_choice"] = chunk_choice
        if ar_choice is not None:
            out["allreduce_choice"] = ar_choice
        if baseline is not None:
            out["megatron_baseline"] = baseline
        if single is not None:
            out["single_layer"] = single
        out["ms_per_layer"] = ms / L
        if probe is not None:
            out["probe"] = probe
        if gpt_mode:
            out["tflops_paper_formula"] = gpt_flops_paper(T, h, a.seq) / (ms * 1e-3) / 1e12
            out["flops_note"] = ("value counts the FLOPs performed (linear 72Th^2 + causal core 7(s+1)Th); "
                                 "tflops_paper_formula uses P:375's 72bsh^2 + 12bs^2h (non-causal core)")
        if plan is not None:
            rk = lambda p: [(r["d1"], r["d2"], r["t_comm"], r["calibrated"]) for r in p["ranked"]]
            out["search"] = {"chosen": plan["chosen"], "ranked": rk(plan),
                             "hcm_only": {"chosen": plan_hcm["chosen"], "ranked": rk(plan_hcm)}}
        emit(out)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
