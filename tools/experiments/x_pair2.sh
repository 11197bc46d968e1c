O=gpurun_out/r02b; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --prf chacha20_et > $O/bench_c3_et.json 2> $O/bench_c3_et.err
timeout 600 python tools/d_sweep.py > $O/d_sweep.jsonl 2>&1
timeout 600 python tools/d_sweep.py --prf chacha20_et > $O/d_sweep_et.jsonl 2>&1
timeout 600 python tools/batch_sweep.py --prf chacha20_et > $O/batch_sweep_c3_et.jsonl 2>&1
timeout 600 python tools/batch_sweep.py > $O/batch_sweep_c3.jsonl 2>&1
