# subtree depth: cost model (default) vs the item-count rule (DPF_M_MODEL=0), batch sweeps + c2 (both schemes)
mkdir -p gpurun_out; O=gpurun_out/mmodel.txt; : > $O
for prf in chacha20 chacha20_et; do
 for shape in "--log-n 22 --D 64" "--log-n 20 --D 256"; do
  echo "== $prf $shape rule" >> $O; DPF_M_MODEL=0 timeout 900 python tools/batch_sweep.py $shape --B 1 2 4 8 16 32 64 --prf $prf --steps 10 2>&1 | grep '^{' >> $O
  echo "== $prf $shape model" >> $O; timeout 900 python tools/batch_sweep.py $shape --B 1 2 4 8 16 32 64 --prf $prf --steps 10 2>&1 | grep '^{' >> $O
 done
done
rm -f gpurun_out/ab.txt
bash tools/ab.sh "--config c2 --prf chacha20_et" "rule:DPF_M_MODEL=0" "model:" "rule2:DPF_M_MODEL=0" "model2:"
bash tools/ab.sh "--config c2 --table rowmajor" "rule:DPF_M_MODEL=0" "model:"
