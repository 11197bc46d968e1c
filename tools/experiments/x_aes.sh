rm -f gpurun_out/ab.txt
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "aes or pbr" > gpurun_out/pytest_aes.txt 2>&1; tail -1 gpurun_out/pytest_aes.txt
bash tools/ab.sh "--prf aes128" "imadhi:" "shr_alu:DPFPIR_LIB=abbuild/lib_pre_aes.so"
bash tools/ab.sh "--config t5 --prf aes128" "imadhi:" "shr_alu:DPFPIR_LIB=abbuild/lib_pre_aes.so"
