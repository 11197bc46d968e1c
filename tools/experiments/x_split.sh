O=gpurun_out/split; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
rm -f gpurun_out/ab.txt
for c in c2 c3 t5; do bash tools/ab.sh "--config $c" "split:" "nosplit:DPF_TAIL_SPLIT=0"; done
for c in c2 c3 t5 c4; do bash tools/ab.sh "--config $c --prf chacha20_et" "split:" "nosplit:DPF_TAIL_SPLIT=0"; done
cp gpurun_out/ab.txt $O/ab.txt
DPF_TAIL_SPLIT=0 timeout 300 python tools/batch_sweep.py --B 8 16 32 64 > $O/bs_nosplit.jsonl 2>&1
timeout 300 python tools/batch_sweep.py --B 8 16 32 64 > $O/bs_split.jsonl 2>&1
