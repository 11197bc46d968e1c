# final round-2 check: full GPU suite, smoke, default bench line, reference arm, ET + AES lines
mkdir -p gpurun_out; O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 600 python bench.py > $O/r02_bench_c3.json 2> $O/r02_bench_c3.err; tail -c 250 $O/r02_bench_c3.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/r02_bench_reference_c3.json 2>&1; tail -c 200 $O/r02_bench_reference_c3.json
timeout 600 python bench.py --config c3 --prf chacha20_et > $O/r02_bench_c3_et.json 2> $O/r02_bench_c3_et.err; tail -c 200 $O/r02_bench_c3_et.json
timeout 600 python bench.py --config c3 --prf aes128 --no-cpu-baseline > $O/aes_check.json 2>&1; tail -c 200 $O/aes_check.json
