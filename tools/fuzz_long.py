"""Long random-shape fuzz on the GPU (not part of the pytest suite): 400 seeded cases
across schemes, IMAD / tcgen05 (pairs, padded D, 4/8-leaf-pair windows) and ragged shards,
bit-exact against the oracle.  python tools/fuzz_long.py [seed]   (r01: seed 11, 400/400 exact)"""
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import synth
from oracle import oracle as orc
from paper_2301_10904_b200 import dpfpir as dp
orc.build()
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 7)
fails = 0; cases = 0
while cases < 400:
    prf = int(rng.choice([1, 2, 3], p=[0.45, 0.1, 0.45]))
    n = int(rng.integers(5 if prf == 3 else 3, 19))
    N = int(rng.integers(max(8, (1 << n) // 3), (1 << n) + 1))
    D = int(rng.choice([4, 32, 64, 96, 128, 256, 384, 512, 1024]))
    B = int(rng.choice([1, 2, 16, 31, 64, 129, 256]))
    if prf == 2 and (n > 11 or B > 64): continue
    if B * N > 40_000_000: continue
    r0 = int(rng.integers(0, N // 2 + 1)); rows = int(rng.integers(1, N - r0 + 1))
    packed = bool(rng.integers(0, 2))
    seed = int(rng.integers(1 << 30))
    T = synth.table(N, D, seed)
    al = synth.alphas(B, N, seed)
    keys = [dp.gen(n, int(a), 1, s, prf=prf)[i % 2] for i, (a, s) in enumerate(zip(al, synth.gen_seeds(B, seed)))]
    ok = [orc.key_from_wire(dp.key_serialize(k)) for k in keys]
    Tsh = T[r0:r0 + rows]; Td = torch.from_numpy(Tsh.view(np.int32)).cuda()
    want = orc.answer_batch(ok, Tsh, row_begin=r0, threads=16)
    got = dp.as_u32(dp.eval_batch_packed(keys, dp.table_pack(Td, r0)) if packed else dp.eval_batch_shard(keys, Td, r0))
    if not np.array_equal(got, want):
        fails += 1; print("FAIL", prf, n, N, D, B, r0, rows, packed, flush=True)
    cases += 1
print("cases", cases, "fails", fails)
