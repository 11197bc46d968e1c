"""Batch-size sweep (the paper's batch/table-size-aware scheduling, P:503-524;
batch-1 latency): ms per batch and the fraction of the binding
roofline -- max(ALU time of the N-1 blocks per key, HBM time of one table
read) -- for B = 1 .. 256 on one table, both contraction paths.
    python tools/batch_sweep.py [--log-n 20] [--D 256] [--B 1 2 4 ...] [--prf chacha20|chacha20_et]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2301_10904_b200 import dpfpir  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--log-n", type=int, default=20)
ap.add_argument("--D", type=int, default=256)
ap.add_argument("--B", type=int, nargs="+", default=[1, 2, 4, 8, 16, 32, 64, 128, 256])
ap.add_argument("--prf", default="chacha20", choices=["chacha20", "chacha20_et"])
ap.add_argument("--steps", type=int, default=10)
args = ap.parse_args()
prf = dpfpir.DPF_PRF_CHACHA20_ET if args.prf == "chacha20_et" else dpfpir.DPF_PRF_CHACHA20
n, D = args.log_n, args.D
N = 1 << n
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json"))) \
    if os.path.exists(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else {}
hbm = float(peaks.get("hbm_gbs", 6650.0)) * 1e9
alu = 148 * 64 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
blocks_per_key = (N - 1) if prf == dpfpir.DPF_PRF_CHACHA20 else (N // 8 - 1)
T = torch.from_numpy(synth.table(N, D, 7).view(np.int32)).cuda()
Tp = dpfpir.table_pack(T)
torch.cuda.synchronize()
for B in args.B:
    al = synth.alphas(B, N, 99 + B)
    keys = [dpfpir.gen(n, int(a), 1, s, prf=prf)[0] for a, s in zip(al, synth.gen_seeds(B, 99 + B))]
    wire = torch.from_numpy(dpfpir.keys_to_wire(keys)).cuda()
    ws = torch.empty(dpfpir.eval_workspace_bytes(B, n, N, D), dtype=torch.uint8, device="cuda")
    out = torch.empty((B, D), dtype=torch.int32, device="cuda")
    for name in ("imad", "tcgen05"):
        if name == "tcgen05":
            try:  # small batches: N = 16 MMA columns, B of them keys (the plan may not fit SMEM)
                dpfpir.eval_batch_wire_packed(wire, n, Tp, out=out, workspace=ws, prf=prf)
            except dpfpir.DpfError:
                continue

        def step():
            if name == "imad":
                dpfpir.eval_batch_wire(wire, n, T, 0, out=out, workspace=ws, prf=prf)
            else:
                dpfpir.eval_batch_wire_packed(wire, n, Tp, out=out, workspace=ws, prf=prf)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        t_alu = 640.0 * B * blocks_per_key / alu
        t_hbm = 4.0 * N * D / hbm
        st = dpfpir.last_eval_stats()
        print(json.dumps({"log_n": n, "D": D, "B": B, "prf": args.prf, "path": name, "ms": round(ms, 4),
                          "qps": round(B / (ms * 1e-3)), "alu_roof_ms": round(t_alu * 1e3, 4),
                          "hbm_roof_ms": round(t_hbm * 1e3, 4),
                          "frac_of_binding_roof": round(max(t_alu, t_hbm) / (ms * 1e-3), 3),
                          "keys_per_tile": st["keys_per_tile"], "items": st["work_items"]}), flush=True)
    del ws
