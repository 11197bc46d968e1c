#!/bin/bash
timeout 600 python tools/shard_sim.py --config c3 > gpurun_out/shard_sim.jsonl 2>&1
timeout 600 python tools/shard_sim.py --config c3 --prf chacha20_et >> gpurun_out/shard_sim.jsonl 2>&1
timeout 900 python tools/shard_sim.py --config c4 --steps 3 >> gpurun_out/shard_sim.jsonl 2>&1
timeout 600 python tools/shard_sim.py --config c4 --prf chacha20_et --steps 5 >> gpurun_out/shard_sim.jsonl 2>&1
timeout 600 python tools/shard_sim.py --config c3 --rank -1 --shards 8 >> gpurun_out/shard_sim.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/shard_sim.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d['config'], d['prf'], d['G'], d['rows'], d['ms_per_gpu'], d['kernel_frac'], d['step_frac'], d['projected_qps'])"
