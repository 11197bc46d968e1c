# AES round 2 with shared lookups (loop unroll 1 / 2) vs the committed kernel; parity gate in each bench run
mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
for cfg in c3 t5; do
bash tools/ab.sh "--config $cfg --prf aes128" "head:DPFPIR_LIB=abbuild/libdpfpir_cur.so" "r2u1:DPFPIR_LIB=abbuild/libdpfpir_aes_r2u1.so" "r2u2:DPFPIR_LIB=abbuild/libdpfpir_aes_r2u2.so" "head2:DPFPIR_LIB=abbuild/libdpfpir_cur.so" "r2u1b:DPFPIR_LIB=abbuild/libdpfpir_aes_r2u1.so" "r2u2b:DPFPIR_LIB=abbuild/libdpfpir_aes_r2u2.so"
done
timeout 900 python -m pytest tests -m gpu -q -x -k "aes or AES" --timeout 600 > gpurun_out/pytest_aes.txt 2>&1; tail -2 gpurun_out/pytest_aes.txt
