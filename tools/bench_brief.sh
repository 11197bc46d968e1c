#!/bin/bash
# usage: tools/bench_brief.sh <config> [extra bench args]  -- one-line summary of a bench run
cfg=$1; shift
python bench.py --config $cfg --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
r=d['roofline']
print('$cfg', 'qps=%.0f'%d['value'], 'ms=%.4f'%d['ms_per_step'], 'kfrac=%.3f'%r['frac'], 'qfrac=%.3f'%r['frac_qps'], 'kshare=%.3f'%r['kernel_share_of_step'], 'e2e=%.0f'%d['e2e']['value'], d['parity'], d['clocks'], d['plan'])"
