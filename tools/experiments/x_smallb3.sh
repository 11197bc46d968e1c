mkdir -p gpurun_out; rm -f gpurun_out/x_smallb3.txt
for env in "" "DPF_FORCE_M=4" "DPF_FORCE_M=5" "DPF_FORCE_M=6"; do
  echo "== $env" >> gpurun_out/x_smallb3.txt
  env $env timeout 300 python tools/batch_sweep.py --B 6 8 12 16 32 >> gpurun_out/x_smallb3.txt 2>&1
  env $env timeout 300 python tools/batch_sweep.py --log-n 22 --D 64 --B 6 12 16 >> gpurun_out/x_smallb3.txt 2>&1
done
