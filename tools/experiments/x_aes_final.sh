# AES bench lines (c3 with the CPU oracle, t5), ncu of the c3 AES fused kernel, full GPU suite
mkdir -p gpurun_out; O=gpurun_out
timeout 900 python bench.py --config c3 --prf aes128 > $O/r02_bench_c3_aes.json 2> $O/r02_bench_c3_aes.err; tail -c 300 $O/r02_bench_c3_aes.json
timeout 900 python bench.py --config t5 --prf aes128 > $O/r02_bench_t5_aes.json 2> $O/r02_bench_t5_aes.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 2 -c 1 -o /tmp/prof_aes python bench.py --config c3 --prf aes128 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/prof_aes.ncu-rep > $O/r02_ncu_c3_aes128.txt 2>&1
python tools/src_hot.py /tmp/prof_aes.ncu-rep 25 > $O/r02_ncu_c3_aes128_src.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_c3_aes.csv python bench.py --config c3 --prf aes128 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
python tools/launch_summary.py $O/launches_c3_aes.csv > $O/r02_launches_c3_aes.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
