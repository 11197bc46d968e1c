#!/bin/bash
DPF_ET_W=2 timeout 300 python -m pytest tests -m gpu -q -x --timeout 120 -k "et" 2>&1 | tail -2
for v in "" "DPF_ET_W=2"; do for c in c3 t5; do echo "== $v $c"; env $v bash tools/bench_brief.sh $c --prf chacha20_et --steps 10 | cut -c1-140; done; done
