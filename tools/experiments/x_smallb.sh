mkdir -p gpurun_out; rm -f gpurun_out/x_smallb.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_shard_dist_gpu.py -m gpu -q -x --timeout 600 > gpurun_out/pytest_smallb.txt 2>&1; tail -3 gpurun_out/pytest_smallb.txt
for env in "" "DPF_TC_SMALLB=0"; do
  echo "== $env" >> gpurun_out/x_smallb.txt
  env $env timeout 300 python tools/batch_sweep.py --B 4 6 8 12 15 16 >> gpurun_out/x_smallb.txt 2>&1
  env $env timeout 300 python tools/batch_sweep.py --log-n 22 --D 64 --B 6 8 12 >> gpurun_out/x_smallb.txt 2>&1
done
