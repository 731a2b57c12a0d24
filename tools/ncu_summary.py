"""Summarise an ncu report (or an ncu --csv launch list) into a committed text file.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep  > profiles/r01_xxx.txt
    python tools/ncu_summary.py --launches gpurun_out/launches.csv > profiles/r01_launches.txt
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "dmma%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("lts__t_sector_hit_rate.pct", "l2hit%"),
    ("smsp__inst_executed.sum", "inst"),
]


def report(path):
    if path.endswith(".csv"):
        raw = open(path).read()
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    kn = hdr.index("Kernel Name")
    cols = [(hdr.index(m), name, units[hdr.index(m)]) for m, name in METRICS if m in hdr]
    print(f"# ncu summary of {path}")
    print("# " + " | ".join(f"{n} [{u}]" for _, n, u in cols))
    for r in rows[2:]:
        name = r[kn].split("(")[0].split("::")[-1]
        print(f"{name:28s} " + " ".join(f"{r[i]:>14s}" for i, _, _ in cols))


def launches(path):
    agg = defaultdict(lambda: [0, 0.0])
    unit = ""
    with open(path) as fh:
        lines = [ln for ln in fh if not ln.startswith("==")]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        unit = r.get("Metric Unit", "")
        name = r["Kernel Name"].split("(")[0].split("::")[-1]
        agg[name][0] += 1
        agg[name][1] += float(r["Metric Value"].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print(f"# launch list {path}: total {tot:.1f} {unit}")
    for name, (cnt, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:32s} launches {cnt:5d}  time {t:12.1f} {unit}  share {100 * t / tot:5.1f}%")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[1])
