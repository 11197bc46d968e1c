timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
bash tools/ab.sh "--config c3 --prf chacha20_et --steps 20 --warmup 5" "et:"
bash tools/ab.sh "--config t5 --prf chacha20_et --steps 20 --warmup 5" "t5et:"
bash tools/ab.sh "--config c4 --prf chacha20_et --steps 5 --warmup 3" "c4et:"
bash tools/ab.sh "--config c2 --prf chacha20_et --steps 50 --warmup 5" "c2et:"
bash tools/ab.sh "--config c3 --steps 10 --warmup 3" "c3:"
bash tools/ab.sh "--config c2 --steps 50 --warmup 5" "c2:"
