mkdir -p gpurun_out
for a in "c2 chacha20" "c2 chacha20_et"; do set -- $a
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python bench.py --config $1 --prf $2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/launch2_$1_$2.csv 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:expand_top -s 3 -c 1 -o /tmp/prof_top \
    python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
ncu -i /tmp/prof_top.ncu-rep --page source --csv --print-source sass > gpurun_out/src_top_c2.csv 2>&1
python tools/ncu_summary.py /tmp/prof_top.ncu-rep > gpurun_out/ncu_top_c2.txt 2>&1
