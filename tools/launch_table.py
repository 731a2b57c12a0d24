"""Per-kernel totals (and optionally every launch) of an ncu --csv launch list."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
tot = OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            name = d["Kernel Name"].split("(")[0].replace("stfem::<unnamed>::", "").replace("void ", "")
            t = float(d["Metric Value"].replace(",", ""))
            if "-v" in sys.argv:
                print(f"{name[:40]:40s} {d['Grid Size']:>16s} {t / 1e3:10.1f} us")
            c, s = tot.get(name, (0, 0.0))
            tot[name] = (c + 1, s + t)
all_t = sum(s for _, s in tot.values())
for k, (c, s) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print(f"{k[:48]:48s} {c:6d} launches {s / 1e6:10.2f} ms {100 * s / all_t:5.1f}%")
