for L in lib_cur lib_swapvar; do
  DPFPIR_LIB=paper_2301_10904_b200/$L.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 2 -c 1 -o /tmp/prof_$L python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/prof_$L.ncu-rep > gpurun_out/ncu_$L.txt 2>&1
  ncu -i /tmp/prof_$L.ncu-rep --page raw --csv > gpurun_out/raw_$L.csv 2>&1
  ncu -i /tmp/prof_$L.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_$L.csv 2>&1
done
