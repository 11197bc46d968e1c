#!/bin/bash
timeout 300 python -m pytest tests -m gpu -q -x --timeout 120 -k "grouped or shapes or deep or wire" 2>&1 | tail -2
timeout 600 python tools/batch_sweep.py --log-n 22 --D 64 --B 1 2 4 8 > gpurun_out/bs.jsonl 2>&1
timeout 600 python tools/batch_sweep.py --B 1 2 4 8 >> gpurun_out/bs.jsonl 2>&1
timeout 900 python tools/codesign_bench.py --batches 1 4 > gpurun_out/c5.jsonl 2>&1; cut -c1-300 gpurun_out/c5.jsonl
cat gpurun_out/bs.jsonl | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d['log_n'],d['D'],d['prf'],d['B'],d['path'],d['ms'],d['qps'],d['alu_roof_ms'],d['hbm_roof_ms'],d['frac_of_binding_roof'],d['keys_per_tile'],d['items'])"
