#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x --timeout 120 2>&1 | tail -4
timeout 200 python __graft_entry__.py smoke 2>&1 | tail -1
for a in c3 t5 c2 "c4 --steps 3" "c3 --prf aes128 --steps 5" "c3 --prf chacha20_et"; do echo "== $a"; timeout 300 bash tools/bench_brief.sh $a --steps 20 2>&1 | cut -c1-90; done
timeout 600 python tools/codesign_bench.py --packed --prf chacha20_et --batches 64 2>&1 | cut -c150-300
