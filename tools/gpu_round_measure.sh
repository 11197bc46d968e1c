#!/bin/bash
# One GPU pass producing the evidence under gpurun_out/ (copied to profiles/ by hand):
# tests, smoke, bench lines per config (standard and early-terminated), D sweeps,
# ncu launch list + text summaries of the fused kernel's full capture.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -c 300 gpurun_out/bench_c3.json
for c in c1 c2 t5 c4; do timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -c 200 gpurun_out/bench_$c.json; done
for c in c3 t5 c2 c4; do timeout 600 python bench.py --config $c --prf chacha20_et > gpurun_out/bench_${c}_et.json 2> gpurun_out/bench_${c}_et.err; tail -c 200 gpurun_out/bench_${c}_et.json; done
timeout 600 python bench.py --table rowmajor --no-cpu-baseline > gpurun_out/bench_c3_rowmajor.json 2>&1
timeout 600 python bench.py --prf aes128 --no-cpu-baseline > gpurun_out/bench_c3_aes.json 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1
timeout 900 python tools/d_sweep.py > gpurun_out/d_sweep.jsonl 2>&1
timeout 900 python tools/d_sweep.py --prf chacha20_et > gpurun_out/d_sweep_et.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
for a in "c3 chacha20" "c3 chacha20_et" "t5 chacha20_et"; do set -- $a
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 2 -c 1 -o /tmp/prof_$1_$2 python bench.py --config $1 --prf $2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/prof_$1_$2.ncu-rep > gpurun_out/ncu_$1_$2.txt 2>&1
  python tools/sass_hot.py /tmp/prof_$1_$2.ncu-rep 25 >> gpurun_out/ncu_$1_$2.txt 2>&1
done
ls -la gpurun_out
timeout 900 python tools/codesign_bench.py > gpurun_out/c5.jsonl 2>&1
timeout 900 python tools/codesign_bench.py --prf chacha20_et > gpurun_out/c5_et.jsonl 2>&1
timeout 900 python tools/codesign_bench.py --packed --prf chacha20_et --batches 16 64 256 1024 > gpurun_out/c5_et_packed.jsonl 2>&1
timeout 600 python tools/batch_sweep.py > gpurun_out/batch_sweep_c3.jsonl 2>&1
timeout 600 python tools/batch_sweep.py --log-n 22 --D 64 > gpurun_out/batch_sweep_22x64.jsonl 2>&1
timeout 600 python tools/batch_sweep.py --prf chacha20_et > gpurun_out/batch_sweep_c3_et.jsonl 2>&1
timeout 600 python tools/shard_sim.py --config c3 > gpurun_out/shard_sim.jsonl 2>&1
timeout 600 python tools/shard_sim.py --config c3 --prf chacha20_et >> gpurun_out/shard_sim.jsonl 2>&1
timeout 900 python tools/shard_sim.py --config c4 --steps 3 >> gpurun_out/shard_sim.jsonl 2>&1
timeout 600 python tools/shard_sim.py --config c4 --prf chacha20_et --steps 5 >> gpurun_out/shard_sim.jsonl 2>&1
ls -la gpurun_out
