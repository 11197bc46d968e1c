mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_eval_tc -s 1 -c 1 -o gpurun_out/prof_d1024 python tools/d_sweep.py --D 1024 --steps 2 > /dev/null 2>&1
ls -la gpurun_out
