# full GPU suite, smoke, AES + c3 bench lines, compute-sanitizer (all four tools) over tools/sanitize_run.py
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 900 python bench.py --config c3 --prf aes128 > gpurun_out/r02_bench_c3_aes.json 2> gpurun_out/r02_bench_c3_aes.err; tail -c 300 gpurun_out/r02_bench_c3_aes.json
timeout 900 python bench.py --config t5 --prf aes128 > gpurun_out/r02_bench_t5_aes.json 2> gpurun_out/r02_bench_t5_aes.err
timeout 900 python bench.py > gpurun_out/r02_bench_c3.json 2> gpurun_out/r02_bench_c3.err; tail -c 300 gpurun_out/r02_bench_c3.json
bash tools/experiments/x_sanitize.sh
