#!/bin/bash
# Round-2 evidence pass (copied to profiles/r02_* by hand): tests, smoke, bench
# lines per config and scheme (incl. the reference arm), launch lists, ncu
# --set full of the fused kernels (-> ncu_traffic entries), sweeps.
mkdir -p gpurun_out/r02
O=gpurun_out/r02
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; tail -c 200 $O/bench_c3.json
for c in c1 c2 t5 c4; do timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
for c in c3 t5 c2 c4; do timeout 600 python bench.py --config $c --prf chacha20_et > $O/bench_${c}_et.json 2> $O/bench_${c}_et.err; done
timeout 900 python bench.py --prf aes128 > $O/bench_c3_aes.json 2> $O/bench_c3_aes.err
timeout 600 python bench.py --table rowmajor --no-cpu-baseline > $O/bench_c3_rowmajor.json 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference_c3.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_c3.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_c3_et.csv python bench.py --prf chacha20_et --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
for a in "c3 chacha20" "c3 chacha20_et" "t5 chacha20_et" "t5 chacha20"; do set -- $a
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 2 -c 1 -o /tmp/prof_$1_$2 python bench.py --config $1 --prf $2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/prof_$1_$2.ncu-rep > $O/ncu_$1_$2.txt 2>&1
  python tools/sass_hot.py /tmp/prof_$1_$2.ncu-rep 25 >> $O/ncu_$1_$2.txt 2>&1
done
timeout 600 python tools/batch_sweep.py > $O/batch_sweep_c3.jsonl 2>&1
timeout 600 python tools/batch_sweep.py --log-n 22 --D 64 > $O/batch_sweep_22x64.jsonl 2>&1
timeout 600 python tools/batch_sweep.py --prf chacha20_et > $O/batch_sweep_c3_et.jsonl 2>&1
timeout 900 python tools/d_sweep.py > $O/d_sweep.jsonl 2>&1
timeout 900 python tools/d_sweep.py --prf chacha20_et > $O/d_sweep_et.jsonl 2>&1
timeout 900 python tools/codesign_bench.py > $O/c5.jsonl 2>&1
timeout 900 python tools/codesign_bench.py --packed --prf chacha20_et --batches 16 64 256 1024 > $O/c5_et_packed.jsonl 2>&1
timeout 900 python tools/codesign_bench.py --scheme pbr --bins 4 > $O/c5_pbr.jsonl 2>&1
timeout 900 python tools/codesign_bench.py --scheme pbr --bins 4 --packed --prf chacha20_et --batches 16 64 256 1024 > $O/c5_pbr_et_packed.jsonl 2>&1
timeout 600 python tools/shard_sim.py --config c3 > $O/shard_sim.jsonl 2>&1
timeout 600 python tools/shard_sim.py --config c3 --prf chacha20_et >> $O/shard_sim.jsonl 2>&1
ls -la $O
