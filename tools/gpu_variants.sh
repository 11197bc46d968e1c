#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -2
for a in "c3" "c3 --prf chacha20_et" "t5 --prf chacha20_et" "c4 --prf chacha20_et --steps 5" "c2 --prf chacha20_et"; do echo "== $a"; bash tools/bench_brief.sh $a --steps 20 2>&1 | cut -c1-100; done
timeout 900 python tools/d_sweep.py --prf chacha20_et > gpurun_out/d_sweep_et.jsonl 2>&1; cut -c1-120 gpurun_out/d_sweep_et.jsonl
timeout 900 python tools/codesign_bench.py --packed --prf chacha20_et --batches 64 1024 2>&1 | cut -c1-300
