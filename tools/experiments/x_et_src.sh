mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 2 -c 1 -o /tmp/prof_et python bench.py --prf chacha20_et --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
ncu -i /tmp/prof_et.ncu-rep --page source --csv --print-source sass > gpurun_out/src_et.csv 2>&1
