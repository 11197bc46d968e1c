rm -f gpurun_out/ab.txt
bash tools/ab.sh "--config c3" "base:" "spin:DPF_LOADER_SPIN=1" "lsleep:DPF_WAIT_SLEEP=2" "base2:" "spin2:DPF_LOADER_SPIN=1"
bash tools/ab.sh "--config t5" "base:" "spin:DPF_LOADER_SPIN=1" "lsleep:DPF_WAIT_SLEEP=2"
