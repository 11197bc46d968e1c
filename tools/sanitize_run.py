"""Small evaluations through every kernel (incl. CTA pairs, which run only
where they widen the MMA: B > 64 at D = 256), for compute-sanitizer:
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
ET = dpfpir.DPF_PRF_CHACHA20_ET
# (n, N, D, B, r0, rows, prf): IMAD and tcgen05 (single CTA, CTA pair, padded D), both schemes, AES
for (n, N, D, B, r0, rows, prf) in ((10, 1000, 64, 40, 0, 1000, 1), (11, 2048, 256, 33, 100, 1500, 1),
                                    (9, 512, 128, 64, 0, 512, 1), (12, 4000, 16, 3, 7, 3000, 1),
                                    (10, 1024, 100, 20, 0, 1024, 1), (12, 4096, 256, 40, 16, 4000, ET),
                                    (10, 1000, 64, 17, 3, 990, ET), (9, 512, 512, 20, 0, 512, 1),
                                    (8, 256, 128, 17, 0, 256, 2), (11, 2048, 256, 6, 8, 2000, 1),
                                    (10, 1024, 128, 4, 0, 1024, 1), (12, 4096, 256, 7, 0, 4096, ET),
                                    (11, 2048, 256, 130, 0, 2048, 1), (11, 2000, 512, 70, 0, 2000, 1),
                                    (11, 2048, 256, 129, 0, 2048, ET)):  # the last three: CTA pairs
    T = synth.table(N, D, n)
    al = synth.alphas(B, N, n)
    keys = [dpfpir.gen(n, int(a), 1, s, prf=prf)[b % 2] for b, (a, s) in enumerate(zip(al, synth.gen_seeds(B, n)))]
    ok_keys = [orc.key_from_wire(dpfpir.key_serialize(k)) for k in keys]
    Tsh = T[r0:r0 + rows]
    want = orc.answer_batch(ok_keys, Tsh, row_begin=r0, threads=8)
    Td = torch.from_numpy(Tsh.view(np.int32)).cuda()
    got = dpfpir.as_u32(dpfpir.eval_batch_shard(keys, Td, r0))
    ok &= np.array_equal(got, want)
    if B >= 16 or (B >= 4 and D % 128 == 0):  # B < 16: the small-batch key mapping (Kr = B, zero MMA columns)
        pk = dpfpir.table_pack(Td, r0)
        ok &= np.array_equal(dpfpir.as_u32(dpfpir.eval_batch_packed(keys, pk)), want)
    lv = dpfpir.as_u32(dpfpir.eval_leaves(keys[:2]))
    ok &= np.array_equal(lv[0], orc.eval_full(ok_keys[0]))
# grouped launches, both schemes
for prf in (1, ET):
    groups, expect = [], []
    for i, (n, N, B) in enumerate(((10, 1000, 3), (12, 4096, 1), (8, 200, 2))):
        T = synth.table(N, 32, 50 + i)
        al = synth.alphas(B, N, 50 + i)
        keys = [dpfpir.gen(n, int(a), 1, s, prf=prf)[0] for a, s in zip(al, synth.gen_seeds(B, 60 + i))]
        wire = torch.from_numpy(dpfpir.keys_to_wire(keys)).cuda()
        out = torch.empty((B, 32), dtype=torch.int32, device="cuda")
        groups.append((wire, n, torch.from_numpy(T.view(np.int32)).cuda(), 0, out))
        expect.append(orc.answer_batch([orc.key_from_wire(dpfpir.key_serialize(k)) for k in keys], T, threads=8))
    dpfpir.eval_grouped(groups, 32, prf=prf)
    torch.cuda.synchronize()
    for g, w in zip(groups, expect):
        ok &= np.array_equal(dpfpir.as_u32(g[4]), w)
# partial batch retrieval (one grouped launch, one group per bin), row-major and packed
N, log_i, D, B = 3000, 9, 128, 3
T = synth.table(N, D, 77)
nb = (N + (1 << log_i) - 1) >> log_i
pairs = [[dpfpir.gen(log_i, (b * 37 + c) % (1 << log_i), 1, synth.gen_seeds(1, 100 * b + c)[0]) for c in range(B)]
         for b in range(nb)]
wire = torch.from_numpy(dpfpir.keys_to_wire([pairs[b][c][0] for b in range(nb) for c in range(B)])).cuda()
Td = torch.from_numpy(T.view(np.int32)).cuda()
want = orc.pbr_answer([[orc.key_from_wire(dpfpir.key_serialize(pairs[b][c][0])) for c in range(B)] for b in range(nb)],
                      T, log_i, threads=8)
for tbl in (Td, dpfpir.table_pack(Td)):
    ok &= np.array_equal(dpfpir.as_u32(dpfpir.eval_pbr(wire, B, log_i, tbl)).reshape(nb, B, D), want)
torch.cuda.synchronize()
print("sanitize_run parity:", ok)
sys.exit(0 if ok else 1)
