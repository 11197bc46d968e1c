# ncu --set full of the AES fused kernel at c3 + launch list (after a plain run)
mkdir -p gpurun_out
O=gpurun_out
timeout 600 python bench.py --config c3 --prf aes128 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > $O/aes_plain.json 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_c3_aes.csv python bench.py --config c3 --prf aes128 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 2 -c 1 -o $O/prof_c3_aes python bench.py --config c3 --prf aes128 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
python tools/ncu_summary.py $O/prof_c3_aes.ncu-rep > $O/ncu_c3_aes128.txt 2>&1
python tools/sass_hot.py $O/prof_c3_aes.ncu-rep 25 >> $O/ncu_c3_aes128.txt 2>&1
python tools/launch_summary.py $O/launches_c3_aes.csv > $O/launches_c3_aes.txt 2>&1
