# c5 co-design workload with the AES-128 PRF (the paper's default PRF): hot split and PBR, IMAD and tcgen05 grouped launches
mkdir -p gpurun_out; O=gpurun_out/r02_codesign_c5_aes.jsonl; : > $O
for scheme in hot pbr; do
  timeout 900 python tools/codesign_bench.py --prf aes128 --scheme $scheme --batches 1 16 64 256 1024 >> $O 2>&1
  timeout 900 python tools/codesign_bench.py --prf aes128 --scheme $scheme --packed --batches 16 64 256 1024 >> $O 2>&1
done
cut -c1-400 $O
