# ET at 2 KiB / 4 KiB entries: forced CTA pairs (N doubles, half the SMEM operand traffic per key) vs unpaired
mkdir -p gpurun_out; O=gpurun_out/et_pair.txt; : > $O
echo "== default" >> $O; timeout 600 python tools/d_sweep.py --D 512 1024 --steps 5 --prf chacha20_et 2>&1 | grep tcgen05 >> $O
echo "== DPF_TC_PAIR=1" >> $O; DPF_TC_PAIR=1 timeout 600 python tools/d_sweep.py --D 512 1024 --steps 5 --prf chacha20_et 2>&1 | grep tcgen05 >> $O
cat $O
