# tcgen05 standard, shallow subtrees: frontier node loaded one item ahead (PrfChachaPf) vs not, c2
mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
bash tools/ab.sh "--config c2" "head:DPFPIR_LIB=abbuild/libdpfpir_cur.so" "pref:" "pref_off:DPF_TC_PREF=0" "head2:DPFPIR_LIB=abbuild/libdpfpir_cur.so" "pref2:" "pref_off2:DPF_TC_PREF=0"
bash tools/ab.sh "--config c3" "head:DPFPIR_LIB=abbuild/libdpfpir_cur.so" "pref:"
timeout 900 python -m pytest tests -m gpu -q -x -k "c2 or grouped or accumulator or small" --timeout 600 > gpurun_out/pytest_pref.txt 2>&1; tail -2 gpurun_out/pytest_pref.txt
