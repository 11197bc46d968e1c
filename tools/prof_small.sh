# ncu captures of the small-batch regime: B = 1 at
# 2^22 x 64 and B = 4 at 2^20 x 256, IMAD kernel (row-major table), plus the
# launch list of each (top BFS + fused).
mkdir -p gpurun_out
for a in "22 64 1" "20 256 4"; do set -- $a
  tag=n$1_d$2_b$3
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv \
    python tools/prof_one.py --log-n $1 --D $2 --B $3 --rowmajor --iters 3 > gpurun_out/launch_$tag.csv 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 2 -c 1 -o /tmp/prof_$tag \
    python tools/prof_one.py --log-n $1 --D $2 --B $3 --rowmajor --iters 3 > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/prof_$tag.ncu-rep > gpurun_out/ncu_$tag.txt 2>&1
  ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv > gpurun_out/raw_$tag.csv 2>&1
done
timeout 600 python tools/batch_sweep.py --log-n 22 --D 64 --B 1 2 4 8 > gpurun_out/bs22.jsonl 2>&1
timeout 600 python tools/batch_sweep.py --B 1 2 4 8 16 > gpurun_out/bs20.jsonl 2>&1
