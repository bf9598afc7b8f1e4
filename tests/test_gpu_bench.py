"""bench.py contract on the GPU (N = 1): one JSON line on stdout with the keys
the driver reads, a roofline object, clocks sampled during the timed region,
libatp kernel launches counted, the e2e number through host buffers, and the
CPU-oracle baseline; small step counts, full default workload."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_json_contract_n1():
    d = _run("--steps", "5", "--warmup", "3", "--cpu-seconds", "2")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "clocks", "gpu_launches", "roofline", "e2e", "cpu_baseline"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] >= 3 and d["value"] > 0
    assert d["gpu_launches"] >= 5 * 12  # at least the 12 GEMMs of every timed step
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic", "peak_burst", "peak_sustained", "peak_rule",
              "gemm_share_of_step"):
        assert k in r, k
    assert r["bound"] == "tensor" and 0 < r["frac"] < 1.5 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-6
    assert r["peak"] in (r["peak_burst"], r["peak_sustained"])
    # the GEMM time comes from a CUPTI trace of the graph-launched step
    kt = d["kernel_trace"]
    assert "error" not in kt, kt
    # (CUPTI GEMM time vs the event-timed step of another pass: equal within noise when GEMMs fill the step)
    assert kt["gemm_launches_per_step"] == 12 and 0.5 < r["gemm_share_of_step"] <= 1.02
    assert d["config"]["hidden"] == 12288 and d["config"]["heads"] == 96  # N=1 default: cfg 5 shape
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["value"] > 0 and c["cores"] >= 1 and c["sample"]
    assert "workload" in d["config"]


def test_bench_n2_shared_gpu():
    """The N>1 bench path (torchrun, NCCL mesh from atp_search, chunk planner,
    graph-captured step, max-over-ranks timing, one JSON line from rank 0) with
    both ranks on the one GPU (--share-gpu: timings meaningless)."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                          "--gpus", "2", "--share-gpu", "--steps", "3", "--warmup", "3", "--hidden", "1024",
                          "--heads", "8", "--batch", "2", "--seq", "1024", "--no-cpu-baseline", "--probe-mib", "4",
                          "--try-fused"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["mesh"] in ([2, 1], [1, 2])
    assert d["search"]["chosen"] == d["config"]["mesh"] and "chunk_choice" in d
    assert d["exposed_comm_ms"] >= 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    # the probe ran and fed the search (calibrated) and the chunk planner (busBW)
    assert "error" not in d["probe"] and d["probe"]["hcm"][0]["ranks"] == 2
    assert d["chunk_choice"]["busbw_source"].startswith("probe") and d["chunk_choice"]["busbw_gbs"] > 0
    assert "hcm_only" in d["search"]
    mb = d.get("megatron_baseline")
    assert mb is None or "error" not in mb, mb
    # N>1 default: a 4-layer stack as one pipeline, with the one-layer call reported beside it
    assert d["config"]["layers"] == 4 and "error" not in d["single_layer"], d.get("single_layer")
    assert abs(d["ms_per_layer"] - d["ms_per_step"] / 4) < 1e-9
    # --try-fused timed the fused GEMM -> reduce-scatter -> all-gather path (CUDA IPC peers) beside NCCL
    ch = d["allreduce_choice"]
    assert "error" not in ch and {"nccl", "fused"} <= set(ch["timed_ms"]), ch


def test_bench_n2_shared_gpu_p2p_disable():
    """The topology-stress path (the paper's IC1 method P:373):
    --p2p-disable sets NCCL_P2P_DISABLE=1 before NCCL init, then the probe ->
    calibrated search runs as usual and the line records the HCM-only and the
    calibrated rankings and the probe's per-pair matrix (2 ranks sharing the
    GPU: the numbers mean nothing, the path is what is checked)."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                          "--gpus", "2", "--share-gpu", "--p2p-disable", "--steps", "3", "--warmup", "3",
                          "--hidden", "1024", "--heads", "8", "--batch", "2", "--seq", "1024", "--layers", "1",
                          "--no-cpu-baseline", "--no-baseline", "--no-e2e", "--probe-mib", "4"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    d = json.loads(lines[-1])
    assert d["config"]["nccl_p2p_disable"] is True and d["probe"]["nccl_p2p_disable"] is True
    assert len(d["probe"]["p2p_matrix_gbps"]) == 2 and d["probe"]["calibration_algbw_gbps"]
    assert d["search"]["chosen"] == d["config"]["mesh"]
    assert {tuple(r[:2]) for r in d["search"]["ranked"]} == {(2, 1), (1, 2)}
    assert {tuple(r[:2]) for r in d["search"]["hcm_only"]["ranked"]} == {(2, 1), (1, 2)}
    assert all(r[3] for r in d["search"]["ranked"]) and not any(r[3] for r in d["search"]["hcm_only"]["ranked"])


def test_bench_gpt_n2_shared_gpu():
    """The full-layer N>1 bench path (--layer gpt: LayerNorm, the attention core
    over the rank's heads with the dim-2 reduce-scatter / all-gather, MLP) under
    torchrun with both ranks on the one GPU: one JSON line from rank 0 with the
    searched mesh, the chunk choice and the paper-formula FLOPs (timings
    meaningless)."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                          "--gpus", "2", "--share-gpu", "--layer", "gpt", "--steps", "3", "--warmup", "3",
                          "--hidden", "1024", "--heads", "8", "--batch", "2", "--seq", "1024", "--no-cpu-baseline",
                          "--probe-mib", "4"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["mesh"] in ([2, 1], [1, 2])
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0 and d["exposed_comm_ms"] >= 0
    assert d["tflops_paper_formula"] > 0
