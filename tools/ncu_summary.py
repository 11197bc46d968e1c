"""Summarise an ncu --set full report of the fused kernel: pipe utilisation,
DRAM traffic, stall reasons and the per-opcode instruction mix.
    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [blocks_per_launch]
"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
blocks = float(sys.argv[2]) if len(sys.argv) > 2 else None


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, units, vals = raw[0], raw[1], raw[2]
m = dict(zip(hdr, vals))
u = dict(zip(hdr, units))
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.per_cycle_active",
        "smsp__inst_executed.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
for k in keys:
    if k in m:
        print("%-62s %s %s" % (k, m[k], u.get(k, "")))
stalls = {k: float(v) for k, v in m.items() if k.startswith("smsp__average_warps_issue_stalled_") and
          k.endswith("_per_issue_active.ratio") and v not in ("", "n/a")}
print("stalls per issue:", ", ".join("%s=%.3f" % (k[len("smsp__average_warps_issue_stalled_"):-len(
    "_per_issue_active.ratio")], v) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:8]))
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source=sass"))))
h = src[1]
ix = {x: i for i, x in enumerate(h)}
c = Counter()
for r in src[2:]:
    s = re.sub(r"^@!?U?P\w+\s+", "", r[ix["Source"]].strip())
    op = s.split()[0] if s else ""
    c[op] += int(r[ix["Instructions Executed"]] or 0)
tot = sum(c.values())
print("warp instructions executed: %d" % tot + (" (%.1f per warp-block)" % (tot / (blocks / 32)) if blocks else ""))
for op, n in c.most_common(14):
    print("  %-34s %12d" % (op, n) + ("  %7.1f per warp-block" % (n / (blocks / 32)) if blocks else ""))
