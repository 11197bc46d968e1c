# final check after the AES 2-stage plan: full GPU suite, smoke, AES bench lines (with the oracle CPU column), c3 default line
mkdir -p gpurun_out; O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 600 python bench.py --config c3 --prf aes128 > $O/r02_bench_c3_aes.json 2> $O/aes.err
timeout 600 python bench.py --config t5 --prf aes128 > $O/r02_bench_t5_aes.json 2>> $O/aes.err
timeout 600 python bench.py > $O/r02_bench_c3.json 2> $O/c3.err; tail -c 150 $O/r02_bench_c3.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_c3_aes.csv python bench.py --config c3 --prf aes128 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
python tools/launch_summary.py $O/launches_c3_aes.csv > $O/r02_launches_c3_aes.txt 2>&1; cat $O/r02_launches_c3_aes.txt
