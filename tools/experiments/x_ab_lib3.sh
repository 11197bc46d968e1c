rm -f gpurun_out/ab.txt
bash tools/ab.sh "--config c3" "r02:DPFPIR_LIB=abbuild/lib_r02.so" "v1:DPFPIR_LIB=abbuild/lib_v1.so DPF_TAIL_SPLIT=0" "v2:DPFPIR_LIB=abbuild/lib_v2.so DPF_TAIL_SPLIT=0" "r02b:DPFPIR_LIB=abbuild/lib_r02.so" "v1b:DPFPIR_LIB=abbuild/lib_v1.so DPF_TAIL_SPLIT=0" "v2b:DPFPIR_LIB=abbuild/lib_v2.so DPF_TAIL_SPLIT=0"
