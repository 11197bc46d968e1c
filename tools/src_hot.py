"""Top CUDA-source lines of an ncu report (-lineinfo builds) by warp
instructions executed and by stall samples (ncu source page, cuda,sass view:
the per-line aggregate rows).
    python tools/src_hot.py report.ncu-rep [n_top]"""
import csv
import io
import os
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
lines, fname, hdr = [], "?", None
for r in rows:
    if r and r[0] == "File Path":
        fname = os.path.basename(r[1])
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[2] == "-":
        lines.append((fname, r))
num = lambda s: float(s) if s.replace(".", "", 1).isdigit() else 0.0
i_n = hdr.index("Instructions Executed")
i_s = hdr.index("Warp Stall Sampling (All Samples)")
for name, col in (("warp instructions executed", i_n), ("stall samples", i_s)):
    tot = sum(num(r[col]) for _, r in lines)
    print("== top source lines by %s (total %.4g)" % (name, tot))
    for f, r in sorted(lines, key=lambda x: -num(x[1][col]))[:ntop]:
        print("%12.4g %5.1f%%  %s:%-5s %s" % (num(r[col]), 100.0 * num(r[col]) / max(tot, 1), f, r[0], r[1].strip()[:80]))
