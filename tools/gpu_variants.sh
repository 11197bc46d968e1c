#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -2
timeout 300 python tools/batch_sweep.py --log-n 22 --D 64 --B 1 2 4 8 2>&1 | cut -c1-110
timeout 300 python tools/batch_sweep.py --B 1 2 4 8 16 2>&1 | cut -c1-110
timeout 600 python tools/codesign_bench.py --batches 1 4 16 2>&1 | cut -c150-260
timeout 600 python tools/codesign_bench.py --prf chacha20_et --batches 1 4 16 64 1024 2>&1 | cut -c150-260
for a in "c3 --table rowmajor" "t5 --table rowmajor" "c1"; do echo "== $a"; bash tools/bench_brief.sh $a --steps 10 2>&1 | cut -c1-100; done
