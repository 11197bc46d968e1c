# small-batch knob sweep after the consumer change + launch list + source profile
mkdir -p gpurun_out; rm -f gpurun_out/x_small2.txt
for env in "" "DPF_NP=16" "DPF_FORCE_M=4" "DPF_FORCE_M=5" "DPF_NP=16 DPF_FORCE_M=3" "DPF_NP=16 DPF_FORCE_M=4"; do
  echo "== $env" >> gpurun_out/x_small2.txt
  env $env timeout 300 python tools/batch_sweep.py --log-n 22 --D 64 --B 1 2 4 >> gpurun_out/x_small2.txt 2>&1
  env $env timeout 300 python tools/batch_sweep.py --log-n 20 --D 256 --B 1 2 4 8 >> gpurun_out/x_small2.txt 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/prof_one.py --log-n 22 --D 64 --B 1 --rowmajor --iters 2 > gpurun_out/launch_b1_v2.csv 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 1 -c 1 -o /tmp/prof_b1 \
    python tools/prof_one.py --log-n 22 --D 64 --B 1 --rowmajor --iters 2 > /dev/null 2>&1
ncu -i /tmp/prof_b1.ncu-rep --page source --csv --print-source sass > gpurun_out/src_b1_v2.csv 2>&1
python tools/ncu_summary.py /tmp/prof_b1.ncu-rep > gpurun_out/ncu_b1_v2.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:expand_top -s 1 -c 1 -o /tmp/prof_top \
    python tools/prof_one.py --log-n 22 --D 64 --B 1 --rowmajor --iters 2 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/prof_top.ncu-rep > gpurun_out/ncu_top_v2.txt 2>&1
