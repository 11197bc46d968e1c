#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -2
for a in c1 c2 "c2 --prf chacha20_et" c3; do echo "== $a"; bash tools/bench_brief.sh $a --steps 30 2>&1 | cut -c1-100; done
