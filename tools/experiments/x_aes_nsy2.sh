# AES: 2-stage y ring buying one more subtree level (shallower top BFS) vs 3 stages (head / DPF_AES_NSY2=0)
mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
for a in "--config c3 --prf aes128" "--config t5 --prf aes128" "--config c2 --prf aes128"; do
  bash tools/ab.sh "$a" "head:DPFPIR_LIB=abbuild/libdpfpir_aes_r2u2.so" "nsy2:" "nsy3:DPF_AES_NSY2=0" "head2:DPFPIR_LIB=abbuild/libdpfpir_aes_r2u2.so" "nsy2b:"
done
timeout 900 python -m pytest tests -m gpu -q -x -k "aes or AES or pbr or grouped" --timeout 600 > gpurun_out/pytest_aes.txt 2>&1; tail -2 gpurun_out/pytest_aes.txt
