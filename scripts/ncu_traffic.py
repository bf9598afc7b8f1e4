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
print(json.dumps(out, indent=1))
