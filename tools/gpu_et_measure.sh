#!/bin/bash
# Measurement pass: gpu tests, smoke, bench lines (standard + early-terminated), ncu text summaries.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -c 300 gpurun_out/bench_c3.json
for c in c3 t5 c2 c4; do timeout 600 python bench.py --config $c --prf chacha20_et > gpurun_out/bench_${c}_et.json 2> gpurun_out/bench_${c}_et.err; tail -c 300 gpurun_out/bench_${c}_et.json; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c3_et.csv python bench.py --prf chacha20_et --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 2 -c 1 -o /tmp/prof_c3_et python bench.py --prf chacha20_et --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ncu_c3_et.log 2>&1
python tools/ncu_summary.py /tmp/prof_c3_et.ncu-rep > gpurun_out/ncu_c3_et_summary.txt 2>&1
python tools/sass_hot.py /tmp/prof_c3_et.ncu-rep 30 > gpurun_out/ncu_c3_et_hot.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:fused -s 2 -c 1 -o /tmp/prof_t5_et python bench.py --config t5 --prf chacha20_et --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/prof_t5_et.ncu-rep > gpurun_out/ncu_t5_et_summary.txt 2>&1
ls -la gpurun_out
