"""A few evaluations of one shape, for ncu:  python tools/prof_one.py --D 512 [--B 256] [--log-n 20] [--rowmajor]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2301_10904_b200 import dpfpir  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--D", type=int, default=256)
ap.add_argument("--B", type=int, default=256)
ap.add_argument("--log-n", type=int, default=20)
ap.add_argument("--rowmajor", action="store_true")
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
n, N = a.log_n, 1 << a.log_n
keys = [dpfpir.gen(n, int(x), 1, s)[0] for x, s in zip(synth.alphas(a.B, N, 1), synth.gen_seeds(a.B, 1))]
wire = torch.from_numpy(dpfpir.keys_to_wire(keys)).cuda()
T = torch.from_numpy(synth.table(N, a.D, 7).view(np.int32)).cuda()
pk = None if a.rowmajor else dpfpir.table_pack(T)
for _ in range(a.iters):
    if pk is None:
        dpfpir.eval_batch_wire(wire, n, T, 0)
    else:
        dpfpir.eval_batch_wire_packed(wire, n, pk)
torch.cuda.synchronize()
print(dpfpir.last_eval_stats())
