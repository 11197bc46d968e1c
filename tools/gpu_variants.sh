#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -2
for a in "c2" "c2 --prf chacha20_et" "c3" "c3 --prf chacha20_et" "t5 --prf chacha20_et" "c1"; do echo "== $a"; bash tools/bench_brief.sh $a --steps 30 | cut -c1-120; done
timeout 600 python tools/batch_sweep.py --log-n 22 --D 64 --B 1 2 4 > gpurun_out/bs.jsonl 2>&1; cut -c1-150 gpurun_out/bs.jsonl
timeout 600 python tools/shard_sim.py --config c3 --prf chacha20_et 2>&1 | cut -c1-160
