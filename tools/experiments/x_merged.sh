# merged limb MMAs (single CTA: 4-6 MMAs per K-chunk/d-tile instead of 10, interleaved limb planes) vs head
mkdir -p gpurun_out; O=gpurun_out/merged.txt; : > $O
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt >> $O
for prf in chacha20_et chacha20; do
  echo "== $prf head" >> $O; DPFPIR_LIB=abbuild/libdpfpir_aes_r2u2.so timeout 600 python tools/d_sweep.py --D 64 256 512 1024 --steps 5 --prf $prf 2>&1 | grep tcgen05 >> $O
  echo "== $prf merged" >> $O; timeout 600 python tools/d_sweep.py --D 64 256 512 1024 --steps 5 --prf $prf 2>&1 | grep tcgen05 >> $O
done
rm -f gpurun_out/ab.txt
for a in "--config t5" "--config c2" "--config c3" "--config c3 --prf chacha20_et" "--config t5 --prf chacha20_et" "--config c2 --prf chacha20_et"; do
  bash tools/ab.sh "$a" "head:DPFPIR_LIB=abbuild/libdpfpir_aes_r2u2.so" "merged:"
done
cat $O | cut -c1-250
