"""Classify compute-sanitizer racecheck hazards (--racecheck-report hazard):
the CTA-pair kernels' paired TMEM allocation writes the TMEM address into the
slot with no kernel PC (reported as a write at +0xffff...), against the CTA's
own tcgen05.alloc.cta_group::2 -- not a data race (the slot is read only after
__syncthreads + barrier.cluster, fused_tc.cuh).  Every other hazard is listed.
    python tools/race_classify.py race.txt"""
import re
import sys

txt = open(sys.argv[1]).read()
blocks = re.findall(r"Error: Potential (\w+) hazard detected.*?\n(.*?)\n(.*?)\n", txt)
alloc, other = 0, []
for kind, w, r in blocks:
    pcless = re.search(r"\+0xf{8,}[0-9a-f]*", w) is not None
    if pcless and "fused_eval_tc_kernel" in w and ", (bool)1" in w.split("fused_eval_tc_kernel")[1][:120]:
        alloc += 1
    else:
        other.append((kind, w.strip(), r.strip()))
print("racecheck hazards: %d total, %d = PC-less paired-TMEM-allocation write (CTA-pair kernels), %d other"
      % (len(blocks), alloc, len(other)))
for o in other[:20]:
    print("  OTHER:", *o)
m = re.search(r"RACECHECK SUMMARY: .*", txt)
print(m.group(0) if m else "no RACECHECK SUMMARY line")
sys.exit(1 if other else 0)
