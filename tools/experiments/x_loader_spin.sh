# T-loader wait: backoff sleep (default) vs spin, at large D (standard and ET)
mkdir -p gpurun_out; O=gpurun_out/loader_spin.txt; : > $O
for prf in chacha20 chacha20_et; do
  echo "== $prf default" >> $O; timeout 600 python tools/d_sweep.py --D 256 512 1024 --steps 3 --prf $prf 2>&1 | grep tcgen05 >> $O
  echo "== $prf DPF_LOADER_SPIN=1" >> $O; DPF_LOADER_SPIN=1 timeout 600 python tools/d_sweep.py --D 256 512 1024 --steps 3 --prf $prf 2>&1 | grep tcgen05 >> $O
done
cat $O
