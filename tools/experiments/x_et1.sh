bash tools/ab.sh "--config c3 --prf chacha20_et --steps 20 --warmup 5" "et_base:" "et_nsy4:DPF_ET_NSY=4" "et_sleep:DPF_PEER_SLEEP=1" "et_both:DPF_ET_NSY=4 DPF_PEER_SLEEP=1" "et_base2:"
bash tools/ab.sh "--config t5 --prf chacha20_et --steps 20 --warmup 5" "t5et_base:" "t5et_nsy4:DPF_ET_NSY=4" "t5et_sleep:DPF_PEER_SLEEP=1"
bash tools/ab.sh "--config c3 --steps 10 --warmup 3" "c3_base:" "c3_sleep:DPF_PEER_SLEEP=1"
