"""Small evaluations through every kernel, for compute-sanitizer:
    compute-sanitizer --tool memcheck python tools/sanitize_run.py
Checks results against the oracle as it goes (exit code 1 on mismatch)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2301_10904_b200 import dpfpir  # noqa: E402

ok = True
for (n, N, D, B, r0, rows) in ((10, 1000, 64, 40, 0, 1000), (11, 2048, 256, 33, 100, 1500), (9, 512, 128, 64, 0, 512),
                               (12, 4000, 16, 3, 7, 3000)):
    T = synth.table(N, D, n)
    al = synth.alphas(B, N, n)
    keys = [dpfpir.gen(n, int(a), 1, s)[b % 2] for b, (a, s) in enumerate(zip(al, synth.gen_seeds(B, n)))]
    ok_keys = [orc.key_from_wire(dpfpir.key_serialize(k)) for k in keys]
    Tsh = T[r0:r0 + rows]
    want = orc.answer_batch(ok_keys, Tsh, row_begin=r0, threads=8)
    Td = torch.from_numpy(Tsh.view(np.int32)).cuda()
    got = dpfpir.as_u32(dpfpir.eval_batch_shard(keys, Td, r0))
    ok &= np.array_equal(got, want)
    if D in (128, 256):
        pk = dpfpir.table_pack(Td, r0)
        ok &= np.array_equal(dpfpir.as_u32(dpfpir.eval_batch_packed(keys, pk)), want)
    lv = dpfpir.as_u32(dpfpir.eval_leaves(keys[:2]))
    ok &= np.array_equal(lv[0], orc.eval_full(ok_keys[0]))
torch.cuda.synchronize()
print("sanitize_run parity:", ok)
sys.exit(0 if ok else 1)
