mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 2 -c 1 -o /tmp/prof_aes2 python bench.py --config c3 --prf aes128 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/prof_aes2.ncu-rep > gpurun_out/r02_ncu_c3_aes128.txt 2>&1
python tools/src_hot.py /tmp/prof_aes2.ncu-rep 25 > gpurun_out/r02_ncu_c3_aes128_src.txt 2>&1
head -8 gpurun_out/r02_ncu_c3_aes128.txt
