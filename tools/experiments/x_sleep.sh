rm -f gpurun_out/ab.txt
bash tools/ab.sh "--config c3 --prf chacha20_et" "base:" "p:DPF_WAIT_SLEEP=1" "l:DPF_WAIT_SLEEP=2" "pl:DPF_WAIT_SLEEP=3" "plm:DPF_WAIT_SLEEP=7" "base2:" "p2:DPF_WAIT_SLEEP=1"
bash tools/ab.sh "--config t5 --prf chacha20_et" "base:" "p:DPF_WAIT_SLEEP=1" "pl:DPF_WAIT_SLEEP=3" "plm:DPF_WAIT_SLEEP=7"
bash tools/ab.sh "--config c3" "base:" "p:DPF_WAIT_SLEEP=1" "pl:DPF_WAIT_SLEEP=3" "plm:DPF_WAIT_SLEEP=7"
