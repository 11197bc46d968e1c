#!/bin/bash
: > gpurun_out/sanitizer.txt
python tools/sanitize_run.py >> gpurun_out/sanitizer.txt 2>&1
for t in memcheck racecheck synccheck initcheck; do
  echo "== $t" >> gpurun_out/sanitizer.txt
  timeout 900 compute-sanitizer --tool $t python tools/sanitize_run.py 2>&1 | tail -3 >> gpurun_out/sanitizer.txt
done
echo "== racecheck detail" >> gpurun_out/sanitizer.txt
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 2 python tools/sanitize_run.py 2>&1 | grep -v "Host Frame\|Saved host" | grep "Error\|Thread\|SUMMARY" | head -12 >> gpurun_out/sanitizer.txt
cat gpurun_out/sanitizer.txt
