O=gpurun_out/split2; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
rm -f gpurun_out/ab.txt
for c in c3 t5 c4; do bash tools/ab.sh "--config $c" "split:" "nosplit:DPF_TAIL_SPLIT=0" "split2:" "nosplit2:DPF_TAIL_SPLIT=0"; done
cp gpurun_out/ab.txt $O/ab.txt
