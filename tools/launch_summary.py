"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, total/mean device time and share of the total.
    python tools/launch_summary.py gpurun_out/launches.csv
"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
agg = OrderedDict()
for r in rows[1:]:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[ix["Kernel Name"]].split("(")[0]
    scale = {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1.0}.get(r[ix["Metric Unit"]], 1.0)
    v = float(r[ix["Metric Value"]].replace(",", "")) * scale
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(v[1] for v in agg.values())
print("%-60s %6s %12s %12s %7s" % ("kernel", "count", "total_us", "mean_us", "share"))
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print("%-60s %6d %12.1f %12.2f %6.1f%%" % (k[:60], n, t / 1e3, t / n / 1e3, 100 * t / tot))
