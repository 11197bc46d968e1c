rm -f gpurun_out/ab.txt
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_20w.txt 2>&1; tail -1 gpurun_out/pytest_20w.txt
bash tools/ab.sh "--config c3" "base:DPFPIR_LIB=abbuild/lib_mq1.so" "w20:DPFPIR_LIB=abbuild/lib_20w.so" "base2:DPFPIR_LIB=abbuild/lib_mq1.so" "w20b:DPFPIR_LIB=abbuild/lib_20w.so"
bash tools/ab.sh "--config t5" "base:DPFPIR_LIB=abbuild/lib_mq1.so" "w20:DPFPIR_LIB=abbuild/lib_20w.so"
bash tools/ab.sh "--config c2" "base:DPFPIR_LIB=abbuild/lib_mq1.so" "w20:DPFPIR_LIB=abbuild/lib_20w.so"
bash tools/ab.sh "--prf aes128" "base:DPFPIR_LIB=abbuild/lib_mq1.so" "w20:DPFPIR_LIB=abbuild/lib_20w.so"
