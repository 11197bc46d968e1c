# round-2 bench lines (the measurement pass's bench calls, after the roofline_of fix)
O=gpurun_out/r02; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
timeout 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; tail -c 200 $O/bench_c3.json
for c in c1 c2 t5 c4; do timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
for c in c3 t5 c2 c4; do timeout 600 python bench.py --config $c --prf chacha20_et > $O/bench_${c}_et.json 2> $O/bench_${c}_et.err; done
timeout 900 python bench.py --prf aes128 > $O/bench_c3_aes.json 2> $O/bench_c3_aes.err
timeout 600 python bench.py --table rowmajor --no-cpu-baseline > $O/bench_c3_rowmajor.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_c3.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_c3_et.csv python bench.py --prf chacha20_et --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
