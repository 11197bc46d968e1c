# A/B of AES T-table variants (same box): committed (k-domain key, unroll 1) vs rot16-domain key (unroll 1 / 2)
mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
cp paper_2301_10904_b200/libdpfpir.so /tmp/cur.so
for cfg in c3 t5; do
bash tools/ab.sh "--config $cfg --prf aes128" "u1_r16:DPFPIR_LIB=abbuild/libdpfpir_tt2_u1.so" "u2_r16:DPFPIR_LIB=abbuild/libdpfpir_tt2_u2.so" "u1_r16b:DPFPIR_LIB=abbuild/libdpfpir_tt2_u1.so" "u2_r16b:DPFPIR_LIB=abbuild/libdpfpir_tt2_u2.so"
done
