#!/bin/bash
DPF_ET_W=2 timeout 600 python -m pytest tests -m gpu -q -x --timeout 120 -k "et_ or fuzz or grouped" 2>&1 | tail -2
for v in "" "DPF_ET_W=2" "" "DPF_ET_W=2"; do for a in "c3 --prf chacha20_et" "t5 --prf chacha20_et"; do echo "== $v $a"; env $v timeout 300 bash tools/bench_brief.sh $a --steps 30 2>&1 | cut -c1-90; done; done
