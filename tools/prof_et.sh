# ncu --set full of the fused tcgen05 kernel (ET and standard, c3) -> CSV pages under gpurun_out/
mkdir -p gpurun_out
for a in "c3 chacha20_et" "c3 chacha20"; do set -- $a
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 2 -c 1 -o /tmp/prof_$1_$2 \
    python bench.py --config $1 --prf $2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
  ncu -i /tmp/prof_$1_$2.ncu-rep --page raw --csv > gpurun_out/raw_$1_$2.csv 2>&1
  ncu -i /tmp/prof_$1_$2.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_$1_$2.csv 2>&1
  python tools/ncu_summary.py /tmp/prof_$1_$2.ncu-rep > gpurun_out/ncu_$1_$2.txt 2>&1
  ls -la gpurun_out/
done
