bash tools/ab.sh "--config c3 --steps 10 --warmup 3" "c3a:" "c3b:" "c3c:"
bash tools/ab.sh "--config t5 --steps 10 --warmup 3" "t5:"
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
