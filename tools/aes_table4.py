"""The paper's Table 4 shape: AES-128 PRF, 2048-bit entries (D = 64
int32 words), tables of 16K, 1M and 4M entries -- GPU throughput and per-batch
latency on the tensor-core path (limb-packed table, T-table AES kernels), the
answers of a few keys checked against the oracle, and the oracle's own rate
on the host (1 thread: one key; all threads: a batch) as the CPU column.  The
paper's batch size for this table is not stated; B is a parameter (default
512, Table 5's batch).
    python tools/aes_table4.py [--B 512] [--log-n 14 20 22] [--cpu-keys 16]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2301_10904_b200 import dpfpir  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=512)
ap.add_argument("--D", type=int, default=64)
ap.add_argument("--log-n", type=int, nargs="+", default=[14, 20, 22])
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--cpu-keys", type=int, default=16, help="keys in the all-threads oracle sample")
ap.add_argument("--cpu-max-s", type=float, default=30.0, help="skip the oracle sample above this estimate")
args = ap.parse_args()
prf = dpfpir.DPF_PRF_AES128
threads = os.cpu_count() or 1
for n in args.log_n:
    N, B, D = 1 << n, args.B, args.D
    T = synth.table(N, D, 4000 + n)
    al = synth.alphas(B, N, 4100 + n)
    keys = [dpfpir.gen(n, int(a), 1, s, prf=prf)[0] for a, s in zip(al, synth.gen_seeds(B, 4200 + n))]
    wire = torch.from_numpy(dpfpir.keys_to_wire(keys)).cuda()
    Tp = dpfpir.table_pack(torch.from_numpy(T.view(np.int32)).cuda())
    out = torch.empty((B, D), dtype=torch.int32, device="cuda")
    ws = torch.empty(dpfpir.eval_workspace_bytes(B, n, N, D), dtype=torch.uint8, device="cuda")

    def step():
        dpfpir.eval_batch_wire_packed(wire, n, Tp, out=out, workspace=ws, prf=prf)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for a, b in evs:
        a.record()
        step()
        b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in evs)
    p50 = ms[len(ms) // 2]
    got = dpfpir.as_u32(out)
    okeys = [orc.key_from_wire(dpfpir.key_serialize(k)) for k in keys]
    sample = [0, B // 2, B - 1]
    exact = bool(np.array_equal(got[sample], orc.answer_batch([okeys[i] for i in sample], T, threads=threads)))
    # the CPU oracle: one key on one thread, then a batch on all threads (bounded)
    t0 = time.perf_counter()
    orc.answer_batch(okeys[:1], T, threads=1)
    t1 = time.perf_counter() - t0
    cpu_mt = None
    if t1 * args.cpu_keys / threads < args.cpu_max_s:
        t0 = time.perf_counter()
        orc.answer_batch(okeys[:args.cpu_keys], T, threads=threads)
        cpu_mt = args.cpu_keys / (time.perf_counter() - t0)
    print(json.dumps({"table": "AES-128 Table 4 shape", "entries": N, "D": D, "entry_bits": 32 * D, "B": B,
                      "gpu_qps": round(B / (p50 * 1e-3)), "gpu_batch_latency_ms": round(p50, 4),
                      "key_bytes": dpfpir.key_wire_size(n) if hasattr(dpfpir, "key_wire_size") else None,
                      "bit_exact_vs_oracle": exact, "oracle_1thread_qps": round(1.0 / t1, 3),
                      "oracle_threads": threads, "oracle_mt_qps": round(cpu_mt, 2) if cpu_mt else None,
                      "plan": dpfpir.last_eval_stats()}), flush=True)
    del T, Tp, ws, out
