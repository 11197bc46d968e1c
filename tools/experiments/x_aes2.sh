rm -f gpurun_out/ab.txt
bash tools/ab.sh "--prf aes128" "imadhi:DPFPIR_LIB=abbuild/lib_aes_imadhi.so" "alu:DPFPIR_LIB=abbuild/lib_aes_alu.so" "imadhi2:DPFPIR_LIB=abbuild/lib_aes_imadhi.so" "alu2:DPFPIR_LIB=abbuild/lib_aes_alu.so"
