bash tools/ab.sh "--config c3 --prf chacha20_et --steps 20 --warmup 5" "et_base:" "et_swap:DPF_ROLE_SWAP=1" "et_w2:DPF_ET_W=2" "et_w2swap:DPF_ET_W=2 DPF_ROLE_SWAP=1"
bash tools/ab.sh "--config t5 --prf chacha20_et --steps 20 --warmup 5" "t5et_base:" "t5et_swap:DPF_ROLE_SWAP=1" "t5et_w2:DPF_ET_W=2"
bash tools/ab.sh "--config c3 --steps 10 --warmup 3" "c3_base:" "c3_swap:DPF_ROLE_SWAP=1"
bash tools/ab.sh "--config t5 --steps 10 --warmup 3" "t5_base:" "t5_swap:DPF_ROLE_SWAP=1"
