mkdir -p gpurun_out
for a in "c2 chacha20" "c2 chacha20_et" "c3 chacha20_et"; do set -- $a
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python bench.py --config $1 --prf $2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/launch_$1_$2.csv 2>&1
done
