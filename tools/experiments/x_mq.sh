rm -f gpurun_out/ab.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "packed" > gpurun_out/pytest_mq.txt 2>&1; tail -1 gpurun_out/pytest_mq.txt
bash tools/ab.sh "--config c3" "base:DPFPIR_LIB=abbuild/lib_base.so" "mq1:DPFPIR_LIB=abbuild/lib_mq1.so" "base2:DPFPIR_LIB=abbuild/lib_base.so" "mq1b:DPFPIR_LIB=abbuild/lib_mq1.so"
bash tools/ab.sh "--config t5" "base:DPFPIR_LIB=abbuild/lib_base.so" "mq1:DPFPIR_LIB=abbuild/lib_mq1.so"
bash tools/ab.sh "--config c2" "base:DPFPIR_LIB=abbuild/lib_base.so" "mq1:DPFPIR_LIB=abbuild/lib_mq1.so"
