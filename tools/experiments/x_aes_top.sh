# AES top BFS with 512-thread CTAs vs 256 (same box), and the AES claimed-size test
mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
bash tools/ab.sh "--config c3 --prf aes128" "top512:" "top256:DPFPIR_LIB=abbuild/libdpfpir_tt2_u2.so" "top512b:" "top256b:DPFPIR_LIB=abbuild/libdpfpir_tt2_u2.so"
bash tools/ab.sh "--config c2 --prf aes128" "top512:" "top256:DPFPIR_LIB=abbuild/libdpfpir_tt2_u2.so"
timeout 900 python -m pytest tests/test_gpu_claimed_sizes.py -m gpu -q --timeout 800 > gpurun_out/pytest_claimed.txt 2>&1; tail -2 gpurun_out/pytest_claimed.txt
