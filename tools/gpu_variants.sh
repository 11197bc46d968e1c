#!/bin/bash
# Scratch A/B driver for tuning passes on the GPU box (gpurun): edit the
# variant list, run, compare the one-line summaries of tools/bench_brief.sh.
# Tuning switches read by libdpfpir (all default off): DPF_NP=8|16,
# DPF_FORCE_M=<m>, DPF_GRID_ALIGN=0|1, DPF_TC_PAIR=0, DPF_TC_W=4,
# DPF_LOADER_SPIN=1, DPF_DEBUG_NOMMA=1 (skips the MMAs: wrong answers).
for v in "" "DPF_TC_W=4"; do
  for a in c3 t5 "c3 --prf chacha20_et"; do
    echo "== $v $a"
    env $v timeout 300 bash tools/bench_brief.sh $a --steps 20 2>&1 | cut -c1-100
  done
done
