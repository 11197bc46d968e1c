rm -f gpurun_out/ab.txt
bash tools/ab.sh "--config c3" "pdl:" "nopdl:DPF_PDL=0" "pdl2:" "nopdl2:DPF_PDL=0" "pdl3:" "nopdl3:DPF_PDL=0"
bash tools/ab.sh "--config t5" "pdl:" "nopdl:DPF_PDL=0" "pdl2:" "nopdl2:DPF_PDL=0"
