#!/bin/bash
for v in "" "DPF_DEBUG_NOMMA=1"; do for a in "c3 --prf chacha20_et" "t5 --prf chacha20_et"; do echo "== $v $a"; env $v bash tools/bench_brief.sh $a --steps 30 2>&1 | cut -c1-90; done; done
