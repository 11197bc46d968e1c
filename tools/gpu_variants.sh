#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
for a in "c3 --prf chacha20_et" "t5 --prf chacha20_et --table packed" "t5 --prf chacha20_et --table rowmajor" "t5 --table packed" "c2 --prf chacha20_et --table packed" "c2 --table packed" "c4 --prf chacha20_et --table packed --steps 5"; do
  echo "== $a"
  bash tools/bench_brief.sh $a --steps 10 2>&1 | tail -1 | cut -c1-230
done
