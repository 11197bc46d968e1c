mkdir -p gpurun_out; rm -f gpurun_out/x_pair.txt
for env in "" "DPF_TC_PAIR=0"; do
  echo "== $env" >> gpurun_out/x_pair.txt
  env $env timeout 600 python tools/d_sweep.py --D 256 512 1024 >> gpurun_out/x_pair.txt 2>&1
  env $env timeout 300 python tools/batch_sweep.py --B 32 64 128 >> gpurun_out/x_pair.txt 2>&1
  env $env timeout 300 python tools/batch_sweep.py --prf chacha20_et --B 128 >> gpurun_out/x_pair.txt 2>&1
  env $env timeout 600 python tools/d_sweep.py --prf chacha20_et --D 256 --B 512 >> gpurun_out/x_pair.txt 2>&1
done
