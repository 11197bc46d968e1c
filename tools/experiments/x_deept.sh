mkdir -p gpurun_out; rm -f gpurun_out/x_deept.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 > gpurun_out/pytest_deept.txt 2>&1; tail -1 gpurun_out/pytest_deept.txt
for env in "" "DPF_ET_DEEPT=0"; do
  echo "== $env" >> gpurun_out/x_deept.txt
  env $env timeout 600 python tools/d_sweep.py --prf chacha20_et --D 512 1024 >> gpurun_out/x_deept.txt 2>&1
done
