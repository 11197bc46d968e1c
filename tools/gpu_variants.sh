#!/bin/bash
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 -k "server" 2>&1 | grep -v "^  " | tail -5
for a in c1 c2 c3 "c2 --prf chacha20_et" "t5"; do echo "== $a"; bash tools/bench_brief.sh $a --steps 30 2>&1 | cut -c1-100; done
