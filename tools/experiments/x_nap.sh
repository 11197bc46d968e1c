# waiting warps: fixed nanosleep naps instead of try_wait spins (T loader, producers on a full y ring)
mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
bash tools/ab.sh "--config c3 --prf chacha20_et" "head:DPFPIR_LIB=abbuild/libdpfpir_cur.so" "nap_off:" "L64:DPF_LOADER_NAP=64" "L200:DPF_LOADER_NAP=200" "P64:DPF_PROD_NAP=64" "L64P64:DPF_LOADER_NAP=64 DPF_PROD_NAP=64" "L200P200:DPF_LOADER_NAP=200 DPF_PROD_NAP=200" "head2:DPFPIR_LIB=abbuild/libdpfpir_cur.so"
bash tools/ab.sh "--config t5 --prf chacha20_et" "head:DPFPIR_LIB=abbuild/libdpfpir_cur.so" "nap_off:" "L64P64:DPF_LOADER_NAP=64 DPF_PROD_NAP=64" "L200P200:DPF_LOADER_NAP=200 DPF_PROD_NAP=200"
bash tools/ab.sh "--config c3" "head:DPFPIR_LIB=abbuild/libdpfpir_cur.so" "nap_off:" "L64P64:DPF_LOADER_NAP=64 DPF_PROD_NAP=64" "P100:DPF_PROD_NAP=100"
