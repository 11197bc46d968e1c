"""Entry-size sweep (the paper's Fig. embedding_entry_size_throughput):
queries/s vs D (int32 words per row) at 2^20 rows, B keys, both contraction
paths where valid (IMAD on the row-major table; tcgen05 on the packed table).
    python tools/d_sweep.py [--B 256] [--log-n 20]
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
import bench  # noqa: E402  (tc_smem_operand_bytes)

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=256)
ap.add_argument("--log-n", type=int, default=20)
ap.add_argument("--D", type=int, nargs="+", default=[16, 32, 64, 128, 256, 512, 1024])
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--prf", default="chacha20", choices=["chacha20", "chacha20_et"])
args = ap.parse_args()
prf = dpfpir.DPF_PRF_CHACHA20_ET if args.prf == "chacha20_et" else dpfpir.DPF_PRF_CHACHA20
n, B = args.log_n, args.B
N = 1 << n
al = synth.alphas(B, N, 99)
keys = [dpfpir.gen(n, int(a), 1, s, prf=prf)[0] for a, s in zip(al, synth.gen_seeds(B, 99))]
blocks_per_key = (N - 1) if prf == dpfpir.DPF_PRF_CHACHA20 else (N // 8 - 1)  # R9 / R20
wire = torch.from_numpy(dpfpir.keys_to_wire(keys)).cuda()
peak = 148 * 64 * 1965e6
smem_peak = 148 * 128 * 1965e6  # B/s: 128 B/clk/SM
for D in args.D:
    T = torch.from_numpy(synth.table(N, D, 7).view(np.int32)).cuda()
    ws = torch.empty(dpfpir.eval_workspace_bytes(B, n, N, D), dtype=torch.uint8, device="cuda")
    out = torch.empty((B, D), dtype=torch.int32, device="cuda")
    paths = [("imad", None)]
    paths.append(("tcgen05", dpfpir.table_pack(T)))
    for name, pk in paths:
        def step():
            if pk is None:
                dpfpir.eval_batch_wire(wire, n, T, 0, out=out, workspace=ws, prf=prf)
            else:
                dpfpir.eval_batch_wire_packed(wire, n, pk, out=out, workspace=ws, prf=prf)
        for _ in range(2):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        st = dpfpir.last_eval_stats()
        # binding roofline: ALU (640 ops per block) or, on the tensor path, the
        # SMEM operand traffic of the limb MMAs at the TMEM-limited MMA N
        bounds = {"alu": 640 * B * blocks_per_key / peak}
        if pk is not None:
            bounds["smem_operands"] = bench.tc_smem_operand_bytes(N, D, B, st["keys_per_tile"],
                                                                  bool((st["kernel_id"] >> 1) & 1)) / smem_peak
        bound = max(bounds, key=bounds.get)
        # table bytes streamed into SMEM per step: once per key tile (N keys, TMEM-limited)
        tstream = (4.0 * N * (((D + 127) // 128 * 128) if pk is not None else D) *
                   -(-B // st["keys_per_tile"]))
        print(json.dumps({"D": D, "entry_bytes": 4 * D, "path": name, "B": B, "log_n": n, "ms": round(ms, 3),
                          "qps": round(B / (ms * 1e-3)), "prf": args.prf,
                          "step_frac_alu": round(bounds["alu"] / (ms * 1e-3), 3),
                          "bound": bound, "bounds_ms": {k: round(v * 1e3, 3) for k, v in bounds.items()},
                          "step_frac_binding": round(bounds[bound] / (ms * 1e-3), 3),
                          "table_stream_gb": round(tstream * 1e-9, 2),
                          "table_stream_tbs": round(tstream / (ms * 1e-3) * 1e-12, 2),
                          "keys_per_tile": st["keys_per_tile"], "frontier_depth": st["frontier_depth"]}), flush=True)
    del T, ws
