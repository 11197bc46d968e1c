mkdir -p gpurun_out; rm -f gpurun_out/x_check3.txt
for env in "" "DPF_STREAM=0"; do
  echo "== $env" >> gpurun_out/x_check3.txt
  env $env timeout 300 python tools/batch_sweep.py --log-n 22 --D 64 --B 1 2 >> gpurun_out/x_check3.txt 2>&1
  env $env timeout 300 python tools/batch_sweep.py --log-n 20 --D 256 --B 1 2 >> gpurun_out/x_check3.txt 2>&1
  env $env timeout 300 python tools/batch_sweep.py --log-n 20 --D 64 --B 1 >> gpurun_out/x_check3.txt 2>&1
  env $env timeout 300 python tools/batch_sweep.py --log-n 24 --D 32 --B 1 >> gpurun_out/x_check3.txt 2>&1
done
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
