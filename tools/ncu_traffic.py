"""Average DRAM traffic per launch of one kernel from an `ncu --set full` report,
merged into profiles/ncu_traffic.json under "<workload>:<family>" (read by
bench.py for roofline.traffic).

    python tools/ncu_traffic.py gpurun_out/syrk_full.ncu-rep C4 syrk [kernel-name regex] [shifts per launch]

The report may also be the raw-page CSV tools/gpu/ncu_cap.sh exports.  "shifts per launch" is
the batch size of the captured run (tools/prof_solve.py --shifts N); bench.py scales the traffic
to its own batch size.
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

rep, workload, family = sys.argv[1:4]
pat = re.compile(sys.argv[4]) if len(sys.argv) > 4 else None
shifts = int(sys.argv[5]) if len(sys.argv) > 5 else None
if rep.endswith(".csv"):
    raw = open(rep).read()
else:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}


def val(r, name):
    v = r[col[name]].replace(",", "")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-6, "us": 1e-3,
             "ms": 1.0, "msecond": 1.0, "usecond": 1e-3, "nsecond": 1e-6}.get(units[col[name]], 1.0)
    return float(v) * scale


if pat is not None:
    data = [r for r in data if pat.search(r[col["Kernel Name"]])]
tot_b, tot_ms = 0.0, 0.0
for r in data:
    tot_b += val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
    tot_ms += val(r, "gpu__time_duration.sum")
n = len(data)
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
cur = json.load(open(path)) if os.path.exists(path) else {}
cur[f"{workload}:{family}"] = {"dram_bytes_per_launch": tot_b / n, "launches_captured": n,
                               "ms_per_launch_under_ncu": tot_ms / n, "report": os.path.basename(rep)}
if shifts:
    cur[f"{workload}:{family}"]["shifts_per_launch"] = shifts
json.dump(cur, open(path, "w"), indent=1)
print(json.dumps(cur[f"{workload}:{family}"]))
