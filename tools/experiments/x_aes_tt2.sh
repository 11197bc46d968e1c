# AES T-table PRF: full GPU suite, smoke, AES bench lines (c3 with the CPU oracle, t5), ncu of the AES fused kernel
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 900 python bench.py --config c3 --prf aes128 > gpurun_out/r02_bench_c3_aes.json 2> gpurun_out/r02_bench_c3_aes.err; tail -c 400 gpurun_out/r02_bench_c3_aes.json
timeout 900 python bench.py --config t5 --prf aes128 > gpurun_out/r02_bench_t5_aes.json 2> gpurun_out/r02_bench_t5_aes.err; tail -c 200 gpurun_out/r02_bench_t5_aes.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_eval_tc_kernel -c 1 -o gpurun_out/ncu_c3_aes -f python bench.py --config c3 --prf aes128 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c3_aes.log 2>&1; tail -2 gpurun_out/ncu_c3_aes.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c3_aes.csv python bench.py --config c3 --prf aes128 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
