# the paper's Table 4 shape with AES-128 (16K / 1M / 4M entries, 2048-bit entries), B = 512 and B = 64
mkdir -p gpurun_out; O=gpurun_out/r02_aes_table4.jsonl; : > $O
timeout 1200 python tools/aes_table4.py --B 512 >> $O 2>&1
timeout 900 python tools/aes_table4.py --B 64 --cpu-keys 4 >> $O 2>&1
cut -c1-300 $O
