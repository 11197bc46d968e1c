rm -f gpurun_out/ab.txt
bash tools/ab.sh "--config c3" "cur:" "r02:DPFPIR_LIB=abbuild/lib_r02.so" "cur2:" "r02b:DPFPIR_LIB=abbuild/lib_r02.so" "nosplit:DPF_TAIL_SPLIT=0"
bash tools/ab.sh "--config c3 --prf chacha20_et" "cur:" "r02:DPFPIR_LIB=abbuild/lib_r02.so"
bash tools/ab.sh "--config t5" "cur:" "r02:DPFPIR_LIB=abbuild/lib_r02.so"
