# B = 1 / 4 knob sweep (NP, m) and a source-level ncu capture of B = 1 (2^22 x 64)
mkdir -p gpurun_out
for env in "" "DPF_NP=16" "DPF_FORCE_M=2" "DPF_FORCE_M=4" "DPF_FORCE_M=5" "DPF_NP=16 DPF_FORCE_M=3" "DPF_NP=16 DPF_FORCE_M=4"; do
  echo "== $env" >> gpurun_out/x_small.txt
  env $env timeout 300 python tools/batch_sweep.py --log-n 22 --D 64 --B 1 4 >> gpurun_out/x_small.txt 2>&1
  env $env timeout 300 python tools/batch_sweep.py --log-n 20 --D 256 --B 1 4 >> gpurun_out/x_small.txt 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 2 -c 1 -o /tmp/prof_b1 \
    python tools/prof_one.py --log-n 22 --D 64 --B 1 --rowmajor --iters 3 > /dev/null 2>&1
ncu -i /tmp/prof_b1.ncu-rep --page source --csv --print-source sass > gpurun_out/src_b1.csv 2>&1
