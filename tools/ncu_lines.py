"""Aggregate an ncu source page (--page source --csv --print-source cuda,sass)
by CUDA source line: stall samples (all / not-issued) and warp instructions.
    python tools/ncu_lines.py src.csv [n_top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg, fpath, hdr = {}, None, None
tot = 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fpath = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0].isdigit():
        continue
    line = int(r[0])
    try:
        s_all = int(r[4] or 0)
        n_inst = int(r[7] or 0)
    except ValueError:
        continue
    key = (fpath, line)
    a = agg.setdefault(key, [0, 0, r[1].strip()[:90]])
    a[0] += s_all
    a[1] += n_inst
    tot += s_all
print("total samples", tot)
for (f, ln), (s, n, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:ntop]:
    print("%6.2f%% %9d %-16s %5d  %s" % (100.0 * s / max(tot, 1), n, f, ln, src))
