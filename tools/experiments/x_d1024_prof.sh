# ncu --set full of the tcgen05 standard kernel at D = 1024 (2^20 rows, B = 256)
mkdir -p gpurun_out; O=gpurun_out
timeout 600 python tools/d_sweep.py --D 1024 --steps 2 > $O/d1024_plain.jsonl 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_eval_tc -s 1 -c 1 -o /tmp/prof_d1024 python tools/d_sweep.py --D 1024 --steps 2 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/prof_d1024.ncu-rep > $O/ncu_d1024.txt 2>&1
python tools/sass_hot.py /tmp/prof_d1024.ncu-rep 30 >> $O/ncu_d1024.txt 2>&1
ncu -i /tmp/prof_d1024.ncu-rep --page raw --csv > $O/ncu_d1024_raw.csv 2>&1
python tools/src_hot.py /tmp/prof_d1024.ncu-rep 30 > $O/ncu_d1024_src.txt 2>&1
