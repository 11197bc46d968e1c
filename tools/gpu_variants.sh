#!/bin/bash
timeout 300 python -m pytest tests -m gpu -q -x --timeout 120 -k "packed or et_ or runs" > gpurun_out/pytest_gpu.txt 2>&1; tail -15 gpurun_out/pytest_gpu.txt
for v in "" "DPF_TC_PAIR=0"; do
for a in "c3" "c3 --prf chacha20_et" "t5 --prf chacha20_et"; do
  echo "== $v $a"
  env $v timeout 300 bash tools/bench_brief.sh $a --steps 10 2>&1 | tail -1 | cut -c1-330
done; done
