"""Per-step DRAM traffic of the GEMM launches from an ncu --set full capture of
ONE bench step (run here on the CPU box):

    python scripts/ncu_traffic.py gpurun_out/prof_step.ncu-rep > profiles/rNN_gemm_traffic.json
"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
h = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
T = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
F = 4 * h


def alg_bytes():
    """Algorithmic bytes of the 12 GEMMs of one DeviceMesh(1,1) step (A + B read once,
    C written once, plus the fused epilogue's extra operand): the op_cost formula."""
    g = lambda M, N, K, out=2, extra=0: 2 * (M * K + N * K) + M * N * (out + extra)
    fwd = [g(T, 3 * h, h), g(T, h, h, extra=2), g(T, F, h, extra=2), g(T, h, F, extra=2)]
    dx = [g(T, F, h, extra=2), g(T, h, F, extra=2), g(T, h, h), g(T, h, 3 * h, extra=2)]
    dw = [g(F, h, T, out=4), g(h, F, T, out=4), g(h, h, T, out=4), g(h, 3 * h, T, out=4)]
    return sum(fwd + dx + dw)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
ix = {k: hdr.index(k) for k in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum")}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
out = {"kernels": [], "gemm_dram_bytes": 0.0, "gemm_launches": 0}
for d in data:
    name = d[ix["Kernel Name"]]
    rd = float(d[ix["dram__bytes_read.sum"]]) * scale[units[ix["dram__bytes_read.sum"]]]
    wr = float(d[ix["dram__bytes_write.sum"]]) * scale[units[ix["dram__bytes_write.sum"]]]
    out["kernels"].append({"kernel": name.split("(")[0][:80], "dram_read": rd, "dram_write": wr})
    if "gemm_sm100" in name:
        out["gemm_dram_bytes"] += rd + wr
        out["gemm_launches"] += 1
out["source"] = rep
out["hidden"], out["tokens"] = h, T
out["gemm_algorithmic_bytes"] = alg_bytes()
out["note"] = ("ncu --set full of one bench step's 12 GEMM launches (DeviceMesh(1,1)); traffic = "
               "dram__bytes_read.sum + dram__bytes_write.sum")
print(json.dumps(out, indent=1))
