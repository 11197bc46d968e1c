# entry-size sweeps (standard and early termination), both contraction paths, current library
mkdir -p gpurun_out
timeout 1200 python tools/d_sweep.py --steps 5 > gpurun_out/r02_d_sweep.jsonl 2>&1
timeout 1200 python tools/d_sweep.py --steps 5 --prf chacha20_et > gpurun_out/r02_d_sweep_et.jsonl 2>&1
cat gpurun_out/r02_d_sweep.jsonl gpurun_out/r02_d_sweep_et.jsonl | cut -c1-150
