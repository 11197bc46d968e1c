# AES byte-3 table addresses on the FMA pipe (IMAD.HI + IMAD) vs the byte permute (head)
mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
for cfg in c3 t5; do
bash tools/ab.sh "--config $cfg --prf aes128" "head:DPFPIR_LIB=abbuild/libdpfpir_aes_r2u2.so" "fma3:" "head2:DPFPIR_LIB=abbuild/libdpfpir_aes_r2u2.so" "fma3b:"
done
timeout 900 python -m pytest tests -m gpu -q -x -k "aes or AES" --timeout 600 > gpurun_out/pytest_aes.txt 2>&1; tail -2 gpurun_out/pytest_aes.txt
