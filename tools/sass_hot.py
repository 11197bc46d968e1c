"""Top stall-sampled SASS lines of an ncu report (source page), with context.
    python tools/sass_hot.py report.ncu-rep [n_top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_src = hdr.index("Source")
i_n = hdr.index("Instructions Executed")
val = lambda r: int(r[i_s]) if r[i_s].isdigit() else 0
tot = sum(val(r) for r in data)
print("total stall samples", tot)
for r in sorted(data, key=lambda r: -val(r))[:ntop]:
    print("%6d %5.1f%%  %s  %-70s %s" % (val(r), 100.0 * val(r) / max(tot, 1), r[0][-5:], r[i_src].strip()[:70], r[i_n]))
