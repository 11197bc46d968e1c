#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -2
for a in c3 t5 c2 "c4 --steps 3" "c3 --prf aes128 --steps 5" "c3 --prf chacha20_et"; do echo "== $a"; bash tools/bench_brief.sh $a --steps 20 2>&1 | cut -c1-90; done
