bash tools/ab.sh "--config c3 --prf chacha20_et --steps 20 --warmup 5" "et_base:" "et_spin:DPF_LOADER_SPIN=1" "et_w2:DPF_ET_W=2" "et_w2spin:DPF_ET_W=2 DPF_LOADER_SPIN=1" "et_w2nomma:DPF_ET_W=2 DPF_DEBUG_NOMMA=1"
bash tools/ab.sh "--config t5 --prf chacha20_et --steps 20 --warmup 5" "t5et_base:" "t5et_w2:DPF_ET_W=2" "t5et_w2spin:DPF_ET_W=2 DPF_LOADER_SPIN=1"
bash tools/ab.sh "--config c3 --steps 10 --warmup 3" "c3_base:" "c3_spin:DPF_LOADER_SPIN=1"
bash tools/ab.sh "--config t5 --steps 10 --warmup 3" "t5_base:"
