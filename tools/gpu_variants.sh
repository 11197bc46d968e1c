#!/bin/bash
timeout 300 python -m pytest tests -m gpu -q -x --timeout 120 -k "grouped" 2>&1 | tail -2
timeout 900 python tools/codesign_bench.py --prf chacha20_et --batches 1 4 16 64 256 1024 > gpurun_out/c5_et.jsonl 2>&1; cut -c1-330 gpurun_out/c5_et.jsonl
