mkdir -p gpurun_out
timeout 300 python tools/batch_sweep.py --log-n 22 --D 64 --B 1 2 4 8 > gpurun_out/bs22_v2.jsonl 2>&1
timeout 300 python tools/batch_sweep.py --B 1 2 4 8 16 > gpurun_out/bs20_v2.jsonl 2>&1
timeout 300 python tools/batch_sweep.py --log-n 20 --D 64 --B 1 2 4 8 > gpurun_out/bs20d64_v2.jsonl 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
