#!/bin/bash
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 -k "packed or et_ or runs" 2>&1 | tail -2
for a in "c3" "c3 --prf chacha20_et" "t5 --prf chacha20_et" "t5" "c3 --prf aes128 --steps 5"; do echo "== $a"; bash tools/bench_brief.sh $a --steps 20 | cut -c1-100; done
