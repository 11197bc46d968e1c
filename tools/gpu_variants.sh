#!/bin/bash
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 -k "grouped" 2>&1 | tail -3
timeout 900 python tools/codesign_bench.py --packed --prf chacha20_et --batches 16 64 256 1024 > gpurun_out/c5_et_packed.jsonl 2>&1; cut -c1-330 gpurun_out/c5_et_packed.jsonl
timeout 900 python tools/codesign_bench.py --packed --batches 16 64 256 > gpurun_out/c5_packed.jsonl 2>&1; cut -c1-330 gpurun_out/c5_packed.jsonl
