mkdir -p gpurun_out; rm -f gpurun_out/x_smallb2.txt
timeout 300 python tools/batch_sweep.py --log-n 22 --D 64 --B 6 8 12 >> gpurun_out/x_smallb2.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 1 -c 1 -o /tmp/prof_b8 \
    python tools/prof_one.py --log-n 20 --D 256 --B 8 --iters 2 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/prof_b8.ncu-rep > gpurun_out/ncu_b8_tc.txt 2>&1
python tools/sass_hot.py /tmp/prof_b8.ncu-rep 20 >> gpurun_out/ncu_b8_tc.txt 2>&1
