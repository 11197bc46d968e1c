mkdir -p gpurun_out; rm -f gpurun_out/x_smallb4.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "small_batch or packed" > gpurun_out/pytest_smallb4.txt 2>&1; tail -2 gpurun_out/pytest_smallb4.txt
timeout 300 python tools/batch_sweep.py --B 2 4 5 6 8 >> gpurun_out/x_smallb4.txt 2>&1
timeout 300 python tools/batch_sweep.py --log-n 22 --D 64 --B 4 5 >> gpurun_out/x_smallb4.txt 2>&1
