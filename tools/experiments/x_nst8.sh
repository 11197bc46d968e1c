# T ring 8 entries (NST=8 build, shallower subtrees) vs 4, large D; and the no-MMA producer bound at D = 1024
mkdir -p gpurun_out; O=gpurun_out/nst8.txt; : > $O
for prf in chacha20 chacha20_et; do
  echo "== $prf NST=4 (current)" >> $O; timeout 600 python tools/d_sweep.py --D 256 512 1024 --steps 3 --prf $prf 2>&1 | grep tcgen05 >> $O
  echo "== $prf NST=8" >> $O; DPFPIR_LIB=abbuild/libdpfpir_nst8.so timeout 600 python tools/d_sweep.py --D 256 512 1024 --steps 3 --prf $prf 2>&1 | grep tcgen05 >> $O
  echo "== $prf NST=4 DPF_DEBUG_NOMMA=1 (wrong answers: producer bound)" >> $O; DPF_DEBUG_NOMMA=1 timeout 600 python tools/d_sweep.py --D 256 1024 --steps 3 --prf $prf 2>&1 | grep tcgen05 >> $O
done
cat $O
