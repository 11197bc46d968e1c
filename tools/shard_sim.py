"""Per-GPU time of rank r's row shard of a config, on ONE GPU (no NCCL):
what each of G GPUs computes in bench.py's row-sharded step.
    python tools/shard_sim.py --config c3 --shards 1 2 4 8 [--table packed|rowmajor]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2301_10904_b200 import dpfpir, shard  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--shards", type=int, nargs="+", default=[1, 2, 4, 8])
ap.add_argument("--table", default="auto")
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--prf", default="chacha20", choices=["chacha20", "chacha20_et"])
ap.add_argument("--rank", type=int, default=0, help="which rank's shard (-1: the last)")
args = ap.parse_args()
prf = dpfpir.DPF_PRF_CHACHA20_ET if args.prf == "chacha20_et" else dpfpir.DPF_PRF_CHACHA20
w = synth.CONFIGS[args.config]
al = synth.alphas(w.B, w.N, w.seed)
seeds = synth.gen_seeds(w.B, w.seed)
keys = [dpfpir.gen(w.log_n, int(a), 1, s, prf=prf)[0] for a, s in zip(al, seeds)]
wire = torch.from_numpy(dpfpir.keys_to_wire(keys)).cuda()
packed = args.table == "packed" or (args.table == "auto" and w.B >= 32)
for G in args.shards:
    r0, rows = shard.row_range(w.N, G, (G - 1) if args.rank < 0 else min(args.rank, G - 1))
    T = torch.from_numpy(synth.table_rows(w.N, w.D, w.seed, r0, r0 + rows).view(np.int32)).cuda()
    Tp = dpfpir.table_pack(T, r0) if packed else None
    out = torch.empty((w.B, w.D), dtype=torch.int32, device="cuda")
    ws = torch.empty(dpfpir.eval_workspace_bytes(w.B, w.log_n, rows, w.D), dtype=torch.uint8, device="cuda")

    def step():
        if packed:
            dpfpir.eval_batch_wire_packed(wire, w.log_n, Tp, out=out, workspace=ws, prf=prf)
        else:
            dpfpir.eval_batch_wire(wire, w.log_n, T, r0, out=out, workspace=ws, prf=prf)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    dpfpir.kernel_timer_begin(args.steps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    kms = dpfpir.kernel_timer_read(args.steps)
    st = dpfpir.last_eval_stats()
    v = 4 if prf == dpfpir.DPF_PRF_CHACHA20_ET else 0
    m = w.log_n - v - st["frontier_depth"]
    blocks = w.B * ((rows >> v) >> m) * ((1 << m) - 1 + ((1 << m) if v else 0))
    frac = 640 * blocks / (sum(kms) / len(kms) * 1e-3) / (148 * 64 * 1965e6)
    g = (G - 1).bit_length()
    per_key = (rows - 1 + g) if not v else (2 * (rows >> v) - 1 + g)
    step_frac = (640 * w.B * per_key / (ms * 1e-3)) / (148 * 64 * 1965e6)
    print(json.dumps({"config": w.name, "prf": args.prf, "G": G, "rows": rows, "ms_per_gpu": round(ms, 4),
                      "kernel_ms": round(sum(kms) / len(kms), 4), "kernel_frac": round(frac, 3),
                      "step_frac": round(step_frac, 3), "projected_qps": round(w.B / (ms * 1e-3)), "plan": st}))
    del T, Tp, ws
