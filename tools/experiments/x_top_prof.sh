# ncu --set full of the top BFS (expand_top_split_kernel) at c2 and c2 ET, and launch lists
mkdir -p gpurun_out; O=gpurun_out
timeout 300 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > $O/c2_plain.json 2>&1 || exit 1
for prf in chacha20 chacha20_et; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:expand_top -s 3 -c 1 -o /tmp/prof_top_c2_$prf python bench.py --config c2 --prf $prf --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/prof_top_c2_$prf.ncu-rep > $O/ncu_top_c2_$prf.txt 2>&1
python tools/sass_hot.py /tmp/prof_top_c2_$prf.ncu-rep 30 >> $O/ncu_top_c2_$prf.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file $O/launches_c2_$prf.csv python bench.py --config c2 --prf $prf --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
python tools/launch_summary.py $O/launches_c2_$prf.csv > $O/launches_c2_$prf.txt 2>&1
done
