#!/bin/bash
for v in "DPF_TC_NSY=3" "DPF_TC_NSY=3 DPF_TC_NST=6" "DPF_TC_NSY=3 DPF_TC_NST=6 DPF_LOADER_SPIN=1" "DPF_TC_NSY=3 DPF_LOADER_SPIN=1"; do
  echo "== $v"
  env $v bash tools/bench_brief.sh c3 --prf chacha20_et --steps 20 2>&1 | tail -1 | cut -c1-200
done
