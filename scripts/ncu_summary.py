"""Summarise ncu output for profiles/ (run here, on the CPU box).

    python scripts/ncu_summary.py full  gpurun_out/prof_gemm.ncu-rep  > profiles/rNN_ncu_gemm.md
    python scripts/ncu_summary.py launches gpurun_out/launches.csv      > profiles/rNN_launches.md
"""
import csv
import io
import subprocess
import sys

FULL_COLS = [
    ("Kernel Name", "kernel"), ("Grid Size", "grid"), ("gpu__time_duration.sum", "us"),
    ("sm__cycles_elapsed.avg.per_second", "SM GHz"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("dram__bytes_read.sum", "DRAM rd"), ("dram__bytes_write.sum", "DRAM wr"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"), ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1 %"),
    ("launch__registers_per_thread", "regs"),
]


def full(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = [(hdr.index(c), name, units[hdr.index(c)]) for c, name in FULL_COLS if c in hdr]
    print("| # | " + " | ".join(f"{n} ({u})" if u else n for _, n, u in idx) + " |")
    print("|" + "---|" * (len(idx) + 1))
    for k, d in enumerate(data):
        cells = []
        for i, n, u in idx:
            v = d[i]
            if n == "kernel":
                v = v.split("(")[0].replace("void ", "").replace("<unnamed>::", "")[:60] + (
                    "<" + d[i].split("<", 1)[1].split(">")[0] + ">" if "<" in d[i] else "")
            cells.append(v)
        print(f"| {k} | " + " | ".join(cells) + " |")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[h], rows[h + 1:]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    ks = [(r[ki], float(r[vi].replace(",", ""))) for r in data if r[mi] == "gpu__time_duration.sum"]
    tot = sum(t for _, t in ks)
    by = {}
    for k, t in ks:
        name = k.split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        name = name.split("<")[0]
        c, s = by.get(name, (0, 0.0))
        by[name] = (c + 1, s + t)
    print(f"{len(ks)} launches, {tot / 1e3:.1f} us total (ncu serialised, cold-cache; compare shares)\n")
    print("| kernel | launches | total us | share |")
    print("|---|---|---|---|")
    for name, (c, s) in sorted(by.items(), key=lambda x: -x[1][1]):
        print(f"| {name} | {c} | {s / 1e3:.1f} | {s / tot:.3f} |")
    print("\n| # | kernel | us |")
    print("|---|---|---|")
    for i, (k, t) in enumerate(ks):
        print(f"| {i} | {k[:90]} | {t / 1e3:.1f} |")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2])
