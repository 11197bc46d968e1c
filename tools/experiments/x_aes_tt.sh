mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "aes or AES or grouped or pbr or leaves" --timeout 600 > gpurun_out/pytest_aes.txt 2>&1; tail -3 gpurun_out/pytest_aes.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
rm -f gpurun_out/ab.txt
bash tools/ab.sh "--config c3 --prf aes128" "tt:" "bs:DPFPIR_LIB=abbuild/libdpfpir_bs.so" "tt2:"
bash tools/ab.sh "--config t5 --prf aes128" "tt:" "bs:DPFPIR_LIB=abbuild/libdpfpir_bs.so"
bash tools/ab.sh "--config c3" "chacha_tt_build:" "chacha_bs_build:DPFPIR_LIB=abbuild/libdpfpir_bs.so"
timeout 300 python bench.py --config c3 --prf aes128 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/aes_c3.json
