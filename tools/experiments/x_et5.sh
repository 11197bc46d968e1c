bash tools/ab.sh "--config c3 --prf chacha20_et --steps 20 --warmup 5" "et_w2spin:DPF_ET_W=2 DPF_LOADER_SPIN=1" "et_w2early:DPF_ET_W=2 DPF_LOADER_SPIN=1 DPF_DEBUG_EARLY_YEMPTY=1" "et_w2nomma:DPF_ET_W=2 DPF_LOADER_SPIN=1 DPF_DEBUG_NOMMA=1" "et_w1early:DPF_LOADER_SPIN=1 DPF_DEBUG_EARLY_YEMPTY=1"
bash tools/ab.sh "--config c3 --steps 10 --warmup 3" "c3_base:" "c3_early:DPF_DEBUG_EARLY_YEMPTY=1"
