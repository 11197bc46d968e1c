# ncu source-line hot spots of the c3 early-termination fused kernel
mkdir -p gpurun_out
timeout 600 python bench.py --config c3 --prf chacha20_et --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/et_plain.json 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 2 -c 1 -o /tmp/prof_et python bench.py --config c3 --prf chacha20_et --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
python tools/src_hot.py /tmp/prof_et.ncu-rep 30 > gpurun_out/ncu_c3_et_src.txt 2>&1
python tools/ncu_summary.py /tmp/prof_et.ncu-rep > gpurun_out/ncu_c3_et.txt 2>&1
