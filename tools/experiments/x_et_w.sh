mkdir -p gpurun_out; rm -f gpurun_out/x_et_w.txt
for env in "" "DPF_ET_W=1"; do
  echo "== $env" >> gpurun_out/x_et_w.txt
  env $env timeout 600 python tools/d_sweep.py --prf chacha20_et --D 256 512 1024 >> gpurun_out/x_et_w.txt 2>&1
  env $env timeout 300 python tools/batch_sweep.py --prf chacha20_et --B 16 32 64 >> gpurun_out/x_et_w.txt 2>&1
done
echo "== DPF_TC_PAIR=0" >> gpurun_out/x_et_w.txt
DPF_TC_PAIR=0 timeout 300 python tools/batch_sweep.py --prf chacha20_et --B 32 64 >> gpurun_out/x_et_w.txt 2>&1
DPF_TC_PAIR=0 timeout 600 python tools/d_sweep.py --prf chacha20_et --D 512 1024 >> gpurun_out/x_et_w.txt 2>&1
