#!/bin/bash
# One GPU pass producing the evidence under gpurun_out/ (copied to profiles/ by hand):
# tests, smoke, bench lines for each config, ncu launch list + full capture of the fused kernel.
set -x
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -c 300 gpurun_out/bench_c3.json
for c in c1 c2 t5 c4; do timeout 600 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -c 200 gpurun_out/bench_$c.json; done
timeout 600 python bench.py --table rowmajor --no-cpu-baseline > gpurun_out/bench_c3_rowmajor.json 2>&1
timeout 600 python bench.py --prf aes128 --no-cpu-baseline > gpurun_out/bench_c3_aes.json 2>&1
timeout 600 python bench.py --config t5 --prf aes128 --no-cpu-baseline > gpurun_out/bench_t5_aes.json 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 2 -c 1 -o gpurun_out/prof_c3 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ncu_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 2 -c 1 -o gpurun_out/prof_t5 python bench.py --config t5 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ncu_t5.log 2>&1
ls -la gpurun_out
