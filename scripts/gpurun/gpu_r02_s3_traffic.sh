# In-step GEMM DRAM traffic of the N=1 bench step (h=12288) with dram metrics only, and the same shapes standalone
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-cupti"
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct"
timeout 900 ncu --metrics $M --clock-control none -k regex:gemm_sm100 --launch-skip 36 --launch-count 12 --csv $B > gpurun_out/traffic_instep.csv 2>/dev/null
timeout 900 ncu --metrics $M --clock-control none -k regex:gemm_sm100 --launch-skip 36 --launch-count 12 --cache-control none --csv $B > gpurun_out/traffic_instep_nocc.csv 2>/dev/null
timeout 600 ncu --metrics $M --clock-control none -k regex:gemm_sm100 --csv python scripts/gemm_bench.py --h 12288 --no-ref --iters 1 > gpurun_out/traffic_standalone.csv 2>/dev/null
for f in traffic_instep traffic_instep_nocc traffic_standalone; do
  echo "== $f"; python - "$f" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(f"gpurun_out/{sys.argv[1]}.csv")) if len(r) > 10]
hdr = rows[0]; ki, mi, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
idi = hdr.index("ID")
sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6, "%": 1}
per = {}
for r in rows[1:]:
    per.setdefault(r[idi], {"k": r[ki][:45]})[r[mi]] = float(r[vi].replace(",", "")) * sc.get(r[ui], 1)
tot = 0
for i, d in per.items():
    rd = d.get("dram__bytes_read.sum", 0) / 1e9; wr = d.get("dram__bytes_write.sum", 0) / 1e9; tot += rd + wr
    print(f"{i:>3} rd {rd:6.2f} GB wr {wr:5.2f} GB  {d.get('gpu__time_duration.sum', 0) / 1e3:8.1f} us  hit {d.get('lts__t_sector_hit_rate.pct', 0):5.1f}%")
print(f"total {tot:.2f} GB over {len(per)} launches")
PY
done
