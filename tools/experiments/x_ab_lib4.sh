rm -f gpurun_out/ab.txt
bash tools/ab.sh "--config c3" "r02:DPFPIR_LIB=abbuild/lib_r02.so" "v3:" "r02b:DPFPIR_LIB=abbuild/lib_r02.so" "v3b:"
bash tools/ab.sh "--config t5" "r02:DPFPIR_LIB=abbuild/lib_r02.so" "v3:"
bash tools/ab.sh "--config c3 --prf chacha20_et" "r02:DPFPIR_LIB=abbuild/lib_r02.so" "v3:"
