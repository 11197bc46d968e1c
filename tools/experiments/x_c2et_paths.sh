mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
bash tools/ab.sh "--config c2 --prf chacha20_et --table packed" "packed:"
bash tools/ab.sh "--config c2 --prf chacha20_et --table rowmajor" "rowmajor:" "rowmajor_np16:DPF_NP=16"
bash tools/ab.sh "--config c2 --prf chacha20_et --table packed" "packed_m:DPF_FORCE_M=2" "packed_m3:DPF_FORCE_M=3"
