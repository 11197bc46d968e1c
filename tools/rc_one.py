import os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import synth
from oracle import oracle as orc
from paper_2301_10904_b200 import dpfpir
ET = dpfpir.DPF_PRF_CHACHA20_ET
which = sys.argv[1]
ok = True
if which.startswith("grouped"):
    prf = ET if which.endswith("et") else 1
    groups, expect = [], []
    for i, (n, N, B) in enumerate(((10, 1000, 3), (12, 4096, 1), (8, 200, 2))):
        T = synth.table(N, 32, 50 + i)
        al = synth.alphas(B, N, 50 + i)
        keys = [dpfpir.gen(n, int(a), 1, s, prf=prf)[0] for a, s in zip(al, synth.gen_seeds(B, 60 + i))]
        wire = torch.from_numpy(dpfpir.keys_to_wire(keys)).cuda()
        out = torch.empty((B, 32), dtype=torch.int32, device="cuda")
        groups.append((wire, n, torch.from_numpy(T.view(np.int32)).cuda(), 0, out))
    dpfpir.eval_grouped(groups, 32, prf=prf)
    print(dpfpir.last_eval_stats())
else:
    n, N, D, B = 12, 4000, 16, 3
    T = synth.table(N, D, n)
    keys = [dpfpir.gen(n, 5, 1, bytes(32))[0] for _ in range(B)]
    Td = torch.from_numpy(T.view(np.int32)).cuda()
    dpfpir.eval_batch_shard(keys, Td, 0)
    print(dpfpir.last_eval_stats())
torch.cuda.synchronize()
