mkdir -p gpurun_out/r02c
O=gpurun_out/r02c
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 2 -c 1 -o /tmp/prof_c3 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/prof_c3.ncu-rep > $O/ncu_c3_chacha20.txt 2>&1
python tools/sass_hot.py /tmp/prof_c3.ncu-rep 25 >> $O/ncu_c3_chacha20.txt 2>&1
ncu -i /tmp/prof_c3.ncu-rep --page source --csv --print-source sass > $O/src_c3.csv 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_c3.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
