"""GPU parity: the CUDA path (through the C ABI) equals the CPU oracle
bit-exactly on the same seeded keys and tables (integer work: the bar is
bit-exact).  Sizes span several work items, windows and
ragged tails; full BASELINE sizes are checked on sampled keys."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def dp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2301_10904_b200 import build as pbuild
    from paper_2301_10904_b200 import dpfpir
    pbuild.build()
    dpfpir.lib()
    return dpfpir


def make_keys(dp, oracle, n, alphas, seed, parties=None, betas=None):
    seeds = synth.gen_seeds(len(alphas), seed)
    keys, okeys = [], []
    for i, (a, s) in enumerate(zip(alphas, seeds)):
        beta = 1 if betas is None else int(betas[i])
        pair = dp.gen(n, int(a), beta, s)
        p = (i % 2) if parties is None else parties[i]
        keys.append(pair[p])
        okeys.append(oracle.key_from_wire(dp.key_serialize(pair[p])))
    return keys, okeys


def to_dev(T):
    return torch.from_numpy(T.view(np.int32)).cuda()


def run_case(dp, oracle, n, N, D, B, seed, row_begin=0, rows=None, betas=None):
    rows = N - row_begin if rows is None else rows
    T = synth.table(N, D, seed)
    al = synth.alphas(B, N, seed)
    keys, okeys = make_keys(dp, oracle, n, al, seed, betas=betas)
    Tsh = T[row_begin:row_begin + rows]
    got = dp.as_u32(dp.eval_batch_shard(keys, to_dev(Tsh), row_begin))
    torch.cuda.synchronize()
    want = oracle.answer_batch(okeys, Tsh, row_begin=row_begin, threads=8)
    np.testing.assert_array_equal(got, want)
    return got


def test_leaves_match_oracle_eval_full(dp, oracle):
    for n, B in ((1, 1), (3, 2), (10, 3), (14, 2)):
        keys, okeys = make_keys(dp, oracle, n, synth.alphas(B, 1 << n, n), n)
        got = dp.as_u32(dp.eval_leaves(keys))
        for b in range(B):
            np.testing.assert_array_equal(got[b], oracle.eval_full(okeys[b]))


def test_c1_exhaustive_two_servers(dp, oracle):
    """Config c1 (BJ:7): 2^10 x 16, every alpha, both servers in-process."""
    w = synth.CONFIGS["c1"]
    T = synth.table(w.N, w.D, w.seed)
    Td = to_dev(T)
    seeds = synth.gen_seeds(w.N, w.seed)
    pairs = [dp.gen(w.log_n, a, 1, seeds[a]) for a in range(w.N)]
    sh = [dp.as_u32(dp.eval_batch([p[x] for p in pairs], Td)) for x in (0, 1)]
    np.testing.assert_array_equal(dp.reconstruct(sh[0], sh[1]), T)          # row alpha for every alpha
    for x in (0, 1):                                                          # bit-exact vs oracle
        ok = [oracle.key_from_wire(dp.key_serialize(p[x])) for p in pairs[:64]]
        np.testing.assert_array_equal(sh[x][:64], oracle.answer_batch(ok, T, threads=8))
    for a in (0, 511, 1023):                                                  # batch 1 (the config's B)
        s0 = dp.as_u32(dp.eval_batch([pairs[a][0]], Td))
        s1 = dp.as_u32(dp.eval_batch([pairs[a][1]], Td))
        np.testing.assert_array_equal(s0[0], sh[0][a])
        np.testing.assert_array_equal(dp.reconstruct(s0, s1)[0], T[a])


@pytest.mark.parametrize("n,N,D,B", [
    (9, 512, 4, 1), (12, 4096, 64, 37), (13, 5000, 32, 64), (11, 2048, 256, 33), (10, 1000, 12, 3),
    (14, 1 << 14, 16, 100), (15, 20000, 128, 40), (8, 256, 1024, 9), (12, 4096, 512, 16), (6, 64, 64, 70),
    (1, 2, 8, 5), (2, 3, 4, 2),
])
def test_parity_shapes(dp, oracle, n, N, D, B):
    run_case(dp, oracle, n, N, D, B, seed=1000 * n + D + B)


def test_parity_c2_full(dp, oracle):
    w = synth.CONFIGS["c2"]
    run_case(dp, oracle, w.log_n, w.N, w.D, w.B, w.seed)
    st = dp.last_eval_stats()
    assert st["prf_blocks"] == w.B * (w.N - 1)  # N-1 blocks per key: optimal work


def test_random_beta_and_wrap(dp, oracle):
    n, N, D, B = 12, 4096, 32, 48
    betas = synth.betas(B, 7, random=True)
    run_case(dp, oracle, n, N, D, B, seed=7, betas=betas)
    # adversarial wrap: all-ones table and beta = 2^32 - 1
    T = np.full((N, D), 0xFFFFFFFF, np.uint32)
    pair = dp.gen(n, 5, 0xFFFFFFFF, bytes(range(32)))
    keys = [pair[0], pair[1], pair[0], pair[1]]
    okeys = [oracle.key_from_wire(dp.key_serialize(k)) for k in keys]
    got = dp.as_u32(dp.eval_batch(keys, to_dev(T)))
    np.testing.assert_array_equal(got, oracle.answer_batch(okeys, T))
    np.testing.assert_array_equal(dp.reconstruct(got[0], got[1]), np.ones(D, np.uint32))


def test_shard_linearity(dp, oracle):
    n, N, D, B = 14, 12345, 64, 40
    T = synth.table(N, D, 9)
    keys, okeys = make_keys(dp, oracle, n, synth.alphas(B, N, 9), 9)
    whole = dp.as_u32(dp.eval_batch(keys, to_dev(T)))
    np.testing.assert_array_equal(whole, oracle.answer_batch(okeys, T, threads=8))
    for cuts in ([0, 4096, 8192, N], [0, 1, 777, 5000, 12000, N], [0, N // 2, N]):
        acc = np.zeros_like(whole)
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            part = dp.as_u32(dp.eval_batch_shard(keys, to_dev(T[lo:hi]), lo))
            np.testing.assert_array_equal(part, oracle.answer_batch(okeys, T[lo:hi], row_begin=lo, threads=8))
            acc += part
        np.testing.assert_array_equal(acc, whole)


def test_wire_and_serve_paths(dp, oracle):
    n, N, D, B = 12, 4096, 64, 32
    T = synth.table(N, D, 11)
    Td = to_dev(T)
    keys, okeys = make_keys(dp, oracle, n, synth.alphas(B, N, 11), 11)
    ref = dp.as_u32(dp.eval_batch(keys, Td))
    wire = torch.from_numpy(dp.keys_to_wire(keys)).cuda()
    np.testing.assert_array_equal(dp.as_u32(dp.eval_batch_wire(wire, n, Td)), ref)
    host = torch.empty((B, D), dtype=torch.int32).pin_memory()
    dp.serve_batch(keys, Td, host)
    np.testing.assert_array_equal(host.numpy().view(np.uint32), ref)
    np.testing.assert_array_equal(ref, oracle.answer_batch(okeys, T, threads=8))
    again = dp.as_u32(dp.eval_batch(keys, Td))  # deterministic
    np.testing.assert_array_equal(again, ref)


def test_full_size_c3_sampled(dp, oracle):
    """BASELINE config c3 (2^20 x 256, B = 256) in the bench's launch
    configuration; the oracle recomputes sampled keys one by one."""
    w = synth.CONFIGS["c3"]
    T = synth.table(w.N, w.D, w.seed)
    al = synth.alphas(w.B, w.N, w.seed)
    seeds = synth.gen_seeds(w.B, w.seed)
    pairs = [dp.gen(w.log_n, int(a), 1, s) for a, s in zip(al, seeds)]
    Td = to_dev(T)
    sh0 = dp.as_u32(dp.eval_batch([p[0] for p in pairs], Td))
    sh1 = dp.as_u32(dp.eval_batch([p[1] for p in pairs], Td))
    st = dp.last_eval_stats()
    assert st["prf_blocks"] == w.B * (w.N - 1)
    np.testing.assert_array_equal(dp.reconstruct(sh0, sh1), T[al.astype(np.int64)])  # every query
    sample = [0, 129, 255]
    ok = [oracle.key_from_wire(dp.key_serialize(pairs[b][b % 2])) for b in sample]
    want = oracle.answer_batch(ok, T, threads=3)
    for i, b in enumerate(sample):
        np.testing.assert_array_equal((sh0, sh1)[b % 2][b], want[i])


# ---------------------------------------------------------------- tcgen05 path

def run_packed_case(dp, oracle, n, N, D, B, seed, row_begin=0, rows=None, T=None):
    rows = N - row_begin if rows is None else rows
    T = synth.table(N, D, seed) if T is None else T
    al = synth.alphas(B, N, seed)
    keys, okeys = make_keys(dp, oracle, n, al, seed)
    Tsh = T[row_begin:row_begin + rows]
    pk = dp.table_pack(to_dev(Tsh), row_begin)
    got = dp.as_u32(dp.eval_batch_packed(keys, pk))
    want = oracle.answer_batch(okeys, Tsh, row_begin=row_begin, threads=8)
    np.testing.assert_array_equal(got, want)
    # the IMAD path on the row-major table agrees too
    np.testing.assert_array_equal(dp.as_u32(dp.eval_batch_shard(keys, to_dev(Tsh), row_begin)), want)
    return got


@pytest.mark.parametrize("n,N,D,B", [
    (12, 4096, 256, 32), (13, 8000, 128, 40), (14, 1 << 14, 256, 64), (10, 1000, 128, 5), (3, 8, 256, 1),
    (11, 2047, 256, 100), (16, 1 << 16, 128, 33), (12, 3000, 384, 40), (11, 2048, 512, 70), (10, 1024, 1024, 20),
    (13, 5000, 640, 17),
])
def test_packed_tc_parity(dp, oracle, n, N, D, B):
    run_packed_case(dp, oracle, n, N, D, B, seed=3000 + n + D + B)


def test_packed_tc_shards_unaligned(dp, oracle):
    n, N, D, B = 13, 6000, 256, 48
    T = synth.table(N, D, 21)
    for lo, hi in ((0, 1001), (1001, 4093), (4093, 6000), (5, 13)):
        run_packed_case(dp, oracle, n, N, D, B, 21, row_begin=lo, rows=hi - lo, T=T)


def test_packed_tc_wraps_mod_2_32(dp, oracle):
    """All-ones limbs over 2^16 leaves overflow every s32 limb accumulator
    many times: exact results prove the accumulation wraps (no saturation)."""
    n, N, D, B = 16, 1 << 16, 128, 32
    T = np.full((N, D), 0xFFFFFFFF, np.uint32)
    run_packed_case(dp, oracle, n, N, D, B, 31, T=T)
    T2 = synth.table(N, D, 5) | np.uint32(0xFF00FF00)
    run_packed_case(dp, oracle, n, N, D, B, 32, T=T2)


def test_packed_tc_c3_sampled(dp, oracle):
    w = synth.CONFIGS["c3"]
    T = synth.table(w.N, w.D, w.seed)
    al = synth.alphas(w.B, w.N, w.seed)
    seeds = synth.gen_seeds(w.B, w.seed)
    pairs = [dp.gen(w.log_n, int(a), 1, s) for a, s in zip(al, seeds)]
    pk = dp.table_pack(to_dev(T))
    sh0 = dp.as_u32(dp.eval_batch_packed([p[0] for p in pairs], pk))
    sh1 = dp.as_u32(dp.eval_batch_packed([p[1] for p in pairs], pk))
    np.testing.assert_array_equal(dp.reconstruct(sh0, sh1), T[al.astype(np.int64)])
    sample = [3, 200]
    ok = [oracle.key_from_wire(dp.key_serialize(pairs[b][0])) for b in sample]
    want = oracle.answer_batch(ok, T, threads=2)
    for i, b in enumerate(sample):
        np.testing.assert_array_equal(sh0[b], want[i])


# ---------------------------------------------------------------- AES-128 PRF (row f1)

def make_aes_keys(dp, oracle, n, alphas, seed):
    keys, okeys = [], []
    for i, (a, s) in enumerate(zip(alphas, synth.gen_seeds(len(alphas), seed))):
        k = dp.gen(n, int(a), 1, s, prf=dp.DPF_PRF_AES128)[i % 2]
        keys.append(k)
        okeys.append(oracle.key_from_wire(dp.key_serialize(k)))
    return keys, okeys


def test_aes_leaves_match_oracle(dp, oracle):
    for n, B in ((1, 2), (4, 3), (10, 2)):
        keys, okeys = make_aes_keys(dp, oracle, n, synth.alphas(B, 1 << n, n), 50 + n)
        got = dp.as_u32(dp.eval_leaves(keys))
        for b in range(B):
            np.testing.assert_array_equal(got[b], oracle.eval_full(okeys[b]))


@pytest.mark.parametrize("n,N,D,B,packed", [
    (10, 1000, 16, 3, False), (12, 4096, 64, 37, False), (13, 5000, 32, 64, False), (9, 512, 4, 1, False),
    (12, 4096, 256, 40, True), (11, 2048, 128, 64, True), (12, 3000, 384, 33, True),
    # small batches on the tensor path (B < MMA N: the Kr key mapping with the AES tables beside it)
    (12, 4096, 256, 5, True), (11, 2048, 128, 1, True), (10, 1000, 64, 12, True), (13, 8000, 512, 2, True),
    # large entries: d-tiles beside the 64 KB of tables (CTA pairs at D = 512, N = 16 at D = 1024)
    (10, 1024, 512, 70, True), (11, 2000, 1024, 40, True),
])
def test_aes_parity(dp, oracle, n, N, D, B, packed):
    T = synth.table(N, D, 600 + n)
    keys, okeys = make_aes_keys(dp, oracle, n, synth.alphas(B, N, 600 + n), 600 + n)
    Td = to_dev(T)
    got = dp.as_u32(dp.eval_batch_packed(keys, dp.table_pack(Td)) if packed else dp.eval_batch(keys, Td))
    np.testing.assert_array_equal(got, oracle.answer_batch(okeys, T, threads=8))


@pytest.mark.parametrize("n,N,r0,rows,D,B", [(13, 8000, 1000, 5000, 256, 40), (12, 4096, 37, 3001, 128, 17),
                                             (11, 2048, 2040, 8, 64, 3)])
def test_aes_packed_shards(dp, oracle, n, N, r0, rows, D, B):
    """AES-128 on the tensor path over row shards with unaligned starts and
    ragged ends (the packed table built from the shard at row_begin r0)."""
    T = synth.table(N, D, 650 + n)
    keys, okeys = make_aes_keys(dp, oracle, n, synth.alphas(B, N, 650 + n), 660 + n)
    Tsh = T[r0:r0 + rows]
    got = dp.as_u32(dp.eval_batch_packed(keys, dp.table_pack(to_dev(Tsh), r0)))
    np.testing.assert_array_equal(got, oracle.answer_batch(okeys, Tsh, row_begin=r0, threads=8))


def test_aes_wire_shard_and_reconstruct(dp, oracle):
    n, N, D, B = 14, 12000, 64, 24
    T = synth.table(N, D, 77)
    al = synth.alphas(B, N, 77)
    pairs = [dp.gen(n, int(a), 1, s, prf=dp.DPF_PRF_AES128) for a, s in zip(al, synth.gen_seeds(B, 77))]
    Td = to_dev(T)
    k0 = [p[0] for p in pairs]
    wire = torch.from_numpy(dp.keys_to_wire(k0)).cuda()
    sh0 = dp.as_u32(dp.eval_batch_wire(wire, n, Td, prf=dp.DPF_PRF_AES128))
    np.testing.assert_array_equal(sh0, dp.as_u32(dp.eval_batch(k0, Td)))
    np.testing.assert_array_equal(dp.keys_to_wire(k0), wire.cpu().numpy())  # caller's device keys untouched
    part = dp.as_u32(dp.eval_batch_shard([p[1] for p in pairs], to_dev(T[5000:]), 5000)) + \
        dp.as_u32(dp.eval_batch_shard([p[1] for p in pairs], to_dev(T[:5000]), 0))
    np.testing.assert_array_equal(dp.reconstruct(sh0, part), T[al.astype(np.int64)])


# ---------------------------------------------------------------- grouped launches (row f2)

@pytest.mark.parametrize("prf", [1, 2])
def test_grouped_equals_per_group_and_oracle(dp, oracle, prf):
    D = 32
    shapes = [(12, 4096, 0, 4096, 5), (9, 300, 0, 300, 17), (14, 9000, 1000, 7000, 40), (1, 2, 0, 2, 3),
              (13, 8192, 0, 8192, 64), (10, 1024, 512, 512, 1)]
    groups, expect = [], []
    for i, (n, N, r0, rows, B) in enumerate(shapes):
        T = synth.table(N, D, 900 + i)
        al = synth.alphas(B, N, 900 + i)
        keys = [dp.gen(n, int(a), 1, s, prf=prf)[(j + i) % 2]
                for j, (a, s) in enumerate(zip(al, synth.gen_seeds(B, 900 + i)))]
        okeys = [oracle.key_from_wire(dp.key_serialize(k)) for k in keys]
        Tsh = T[r0:r0 + rows]
        wire = torch.from_numpy(dp.keys_to_wire(keys)).cuda()
        out = torch.empty((B, D), dtype=torch.int32, device="cuda")
        groups.append((wire, n, to_dev(Tsh), r0, out))
        expect.append(oracle.answer_batch(okeys, Tsh, row_begin=r0, threads=8))
    dp.eval_grouped(groups, D, prf=prf)
    torch.cuda.synchronize()
    for (wire, n, Td, r0, out), want in zip(groups, expect):
        np.testing.assert_array_equal(dp.as_u32(out), want)
        np.testing.assert_array_equal(dp.as_u32(dp.eval_batch_wire(wire, n, Td, r0, prf=prf)), want)


def test_deep_domains_small_shards(dp, oracle):
    """log_n up to 32 with a small shard anywhere in the domain: the top BFS
    descends the path to the shard (SMEM levels + grid-wide levels)."""
    D, B = 16, 6
    for n, r0, rows in ((28, (1 << 27) + 12345, 3000), (32, (1 << 32) - 4096, 4096), (24, 0, 1000),
                        (31, 1 << 30, 2048)):
        T = synth.table(rows, D, n)
        al = [r0 + (i * 997) % rows for i in range(B)]
        pairs = [dp.gen(n, a, 1, s) for a, s in zip(al, synth.gen_seeds(B, n))]
        Td = to_dev(T)
        s0 = dp.as_u32(dp.eval_batch_shard([p[0] for p in pairs], Td, r0))
        s1 = dp.as_u32(dp.eval_batch_shard([p[1] for p in pairs], Td, r0))
        np.testing.assert_array_equal(dp.reconstruct(s0, s1), T[[a - r0 for a in al]])
        # spot-check one key against the oracle's point evaluations over the shard
        ok = oracle.key_from_wire(dp.key_serialize(pairs[0][0]))
        y = np.array([oracle.eval_point(ok, r0 + j) for j in range(rows)], np.uint32)
        np.testing.assert_array_equal(s0[0], oracle.contract(y, T))


# ---------------------------------------------------------------- early-terminated leaves (row f4, R20)

ET = 3


def make_et_keys(dp, oracle, n, alphas, seed, betas=None):
    keys, okeys = [], []
    for i, (a, s) in enumerate(zip(alphas, synth.gen_seeds(len(alphas), seed))):
        beta = 1 if betas is None else int(betas[i])
        k = dp.gen(n, int(a), beta, s, prf=ET)[i % 2]
        keys.append(k)
        okeys.append(oracle.key_from_wire(dp.key_serialize(k)))
    return keys, okeys


def test_et_leaves_match_oracle(dp, oracle):
    for n, B in ((5, 2), (6, 3), (12, 2), (16, 1)):
        keys, okeys = make_et_keys(dp, oracle, n, synth.alphas(B, 1 << n, n), 70 + n)
        got = dp.as_u32(dp.eval_leaves(keys))
        for b in range(B):
            np.testing.assert_array_equal(got[b], oracle.eval_full(okeys[b]))


@pytest.mark.parametrize("n,N,D,B", [
    (5, 32, 4, 1), (6, 50, 16, 3), (9, 512, 64, 33), (12, 4096, 64, 37), (13, 5000, 32, 64), (10, 1000, 12, 7),
    (14, 1 << 14, 256, 100), (15, 20000, 128, 40), (8, 256, 1024, 9), (16, 1 << 16, 64, 64), (11, 2047, 8, 2),
])
def test_et_parity_imad(dp, oracle, n, N, D, B):
    T = synth.table(N, D, 4000 + n + D)
    keys, okeys = make_et_keys(dp, oracle, n, synth.alphas(B, N, 4000 + n), 4000 + n + B,
                               betas=synth.betas(B, n, random=True))
    got = dp.as_u32(dp.eval_batch(keys, to_dev(T)))
    np.testing.assert_array_equal(got, oracle.answer_batch(okeys, T, threads=8))


@pytest.mark.parametrize("n,N,D,B", [
    (12, 4096, 256, 32), (13, 8000, 128, 40), (14, 1 << 14, 256, 64), (10, 1000, 128, 5), (5, 32, 256, 1),
    (11, 2047, 256, 100), (16, 1 << 16, 128, 33), (12, 3000, 384, 40), (11, 2048, 512, 70), (10, 1024, 1024, 20),
    (6, 64, 128, 3),
])
def test_et_parity_tc(dp, oracle, n, N, D, B):
    T = synth.table(N, D, 5000 + n + D)
    keys, okeys = make_et_keys(dp, oracle, n, synth.alphas(B, N, 5000 + n), 5000 + n + B)
    Td = to_dev(T)
    got = dp.as_u32(dp.eval_batch_packed(keys, dp.table_pack(Td)))
    want = oracle.answer_batch(okeys, T, threads=8)
    np.testing.assert_array_equal(got, want)
    np.testing.assert_array_equal(dp.as_u32(dp.eval_batch(keys, Td)), want)


def test_et_shards_wire_and_reconstruct(dp, oracle):
    n, N, D, B = 14, 12345, 128, 40
    T = synth.table(N, D, 88)
    al = synth.alphas(B, N, 88)
    pairs = [dp.gen(n, int(a), 1, s, prf=ET) for a, s in zip(al, synth.gen_seeds(B, 88))]
    Td = to_dev(T)
    k0, k1 = [p[0] for p in pairs], [p[1] for p in pairs]
    whole = dp.as_u32(dp.eval_batch(k0, Td))
    ok = [oracle.key_from_wire(dp.key_serialize(k)) for k in k0[:8]]
    np.testing.assert_array_equal(whole[:8], oracle.answer_batch(ok, T, threads=8))
    wire = torch.from_numpy(dp.keys_to_wire(k0)).cuda()
    np.testing.assert_array_equal(dp.as_u32(dp.eval_batch_wire(wire, n, Td, prf=ET)), whole)
    pk = dp.table_pack(Td)
    np.testing.assert_array_equal(dp.as_u32(dp.eval_batch_wire_packed(wire, n, pk, prf=ET)), whole)
    for cuts in ([0, 4096, 8192, N], [0, 1, 777, 5000, 12000, N], [0, 7, 9, N]):  # cuts inside final nodes
        acc = np.zeros_like(whole)
        acc_tc = np.zeros_like(whole)
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            acc += dp.as_u32(dp.eval_batch_shard(k0, to_dev(T[lo:hi]), lo))
            acc_tc += dp.as_u32(dp.eval_batch_packed(k0, dp.table_pack(to_dev(T[lo:hi]), lo)))
        np.testing.assert_array_equal(acc, whole)
        np.testing.assert_array_equal(acc_tc, whole)
    sh1 = dp.as_u32(dp.eval_batch(k1, Td))
    np.testing.assert_array_equal(dp.reconstruct(whole, sh1), T[al.astype(np.int64)])


def test_et_c3_full_size_sampled(dp, oracle):
    """Config c3's shape (2^20 x 256, B = 256) with ET keys in the bench's launch
    configuration (tcgen05 path); every query reconstructs, sampled keys equal
    the oracle, and the device computes N/8 - 1 blocks per key."""
    w = synth.CONFIGS["c3"]
    T = synth.table(w.N, w.D, w.seed)
    al = synth.alphas(w.B, w.N, w.seed)
    pairs = [dp.gen(w.log_n, int(a), 1, s, prf=ET) for a, s in zip(al, synth.gen_seeds(w.B, w.seed))]
    pk = dp.table_pack(to_dev(T))
    sh0 = dp.as_u32(dp.eval_batch_packed([p[0] for p in pairs], pk))
    assert dp.last_eval_stats()["prf_blocks"] == w.B * (w.N // 8 - 1)
    sh1 = dp.as_u32(dp.eval_batch_packed([p[1] for p in pairs], pk))
    np.testing.assert_array_equal(dp.reconstruct(sh0, sh1), T[al.astype(np.int64)])
    sample = [0, 77, 255]
    want = oracle.answer_batch([oracle.key_from_wire(dp.key_serialize(pairs[b][0])) for b in sample], T, threads=3)
    for i, b in enumerate(sample):
        np.testing.assert_array_equal(sh0[b], want[i])


@pytest.mark.parametrize("n,N,D,B,prf,packed", [
    (14, 1 << 14, 64, 37 * 32, 1, False),   # IMAD: 37 key tiles, aligned grid of 148
    (14, (1 << 14) - 5, 128, 256, 1, True),   # tcgen05: 4 key tiles, ragged N
    (16, 60000, 256, 256, 3, True),         # early termination, tcgen05
    (18, 250000, 64, 64, 3, False),         # early termination, IMAD: 2 key tiles, ragged N
])
def test_accumulator_runs_across_items(dp, oracle, n, N, D, B, prf, packed):
    """A CTA keeps its accumulators across consecutive items of one key tile
    and flushes once per run (run_continues): many items per CTA, exact."""
    plan = dp.eval_plan(B, n, N, D, prf=prf, packed=packed)
    assert plan["work_items"] > plan["grid"]
    n_kt = -(-B // plan["keys_per_tile"])
    assert plan["grid"] % n_kt == 0  # every CTA stays on one key tile
    T = synth.table(N, D, 9100 + n)
    al = synth.alphas(B, N, 9100 + n)
    if prf == 3:
        keys, okeys = make_et_keys(dp, oracle, n, al, 9200 + n)
    else:
        keys, okeys = make_keys(dp, oracle, n, al, 9200 + n)
    Td = to_dev(T)
    got = dp.as_u32(dp.eval_batch_packed(keys, dp.table_pack(Td)) if packed else dp.eval_batch(keys, Td))
    assert dp.last_eval_stats()["grid"] == plan["grid"]
    np.testing.assert_array_equal(got, oracle.answer_batch(okeys, T, threads=16))


@pytest.mark.parametrize("n,N,D,B,prf", [
    (12, 4096, 64, 130, 1), (11, 2000, 4, 3, 1), (12, 4000, 100, 70, 1), (10, 1024, 192, 40, 1),
    (11, 2047, 1000, 17, 1), (13, 1 << 13, 64, 128, 3), (12, 3001, 36, 129, 3), (10, 1000, 320, 33, 2),
])
def test_packed_tc_padded_columns(dp, oracle, n, N, D, B, prf):
    """tcgen05 path for D not a multiple of 128: the packed table is padded
    with zero columns to whole 128-column d-tiles (Kt = 128 keys at D <= 128)."""
    T = synth.table(N, D, 9300 + D)
    al = synth.alphas(B, N, 9300 + n)
    if prf == 3:
        keys, okeys = make_et_keys(dp, oracle, n, al, 9400 + n)
    else:
        seeds = synth.gen_seeds(B, 9400 + n)
        keys, okeys = [], []
        for i, (a, s) in enumerate(zip(al, seeds)):
            k = dp.gen(n, int(a), 1, s, prf=prf)[i % 2]
            keys.append(k)
            okeys.append(oracle.key_from_wire(dp.key_serialize(k)))
    Tp = dp.table_pack(to_dev(T))
    got = dp.as_u32(dp.eval_batch_packed(keys, Tp))
    np.testing.assert_array_equal(got, oracle.answer_batch(okeys, T, threads=16))


@pytest.mark.parametrize("D", [32, 64])
def test_grouped_small_batches_streaming(dp, oracle, D):
    """Co-design at inference batch 1 (row f2): 1-2 keys per group (shared key
    tile 1 -> streaming regime, one window per subtree), tiny and ragged hot
    tables next to large full ones, deep frontiers (> 10 top levels)."""
    shapes = [(18, 1 << 18, 0, 1 << 18, 1), (15, 26215, 0, 26215, 2), (12, 409, 0, 409, 2), (16, 1 << 16, 0, 1 << 16, 1),
              (9, 300, 0, 300, 1), (17, 100000, 3, 99990, 2)]
    groups, expect = [], []
    for i, (n, N, r0, rows, B) in enumerate(shapes):
        T = synth.table(N, D, 950 + i)
        al = synth.alphas(B, N, 950 + i)
        keys = [dp.gen(n, int(a), 1, s)[(j + i) % 2] for j, (a, s) in enumerate(zip(al, synth.gen_seeds(B, 950 + i)))]
        okeys = [oracle.key_from_wire(dp.key_serialize(k)) for k in keys]
        Tsh = T[r0:r0 + rows]
        wire = torch.from_numpy(dp.keys_to_wire(keys)).cuda()
        out = torch.empty((B, D), dtype=torch.int32, device="cuda")
        groups.append((wire, n, to_dev(Tsh), r0, out))
        expect.append(oracle.answer_batch(okeys, Tsh, row_begin=r0, threads=8))
    dp.eval_grouped(groups, D)
    torch.cuda.synchronize()
    for (wire, n, Td, r0, out), want in zip(groups, expect):
        np.testing.assert_array_equal(dp.as_u32(out), want)


@pytest.mark.parametrize("kt_keys", [1, 40])
def test_grouped_early_termination(dp, oracle, kt_keys):
    """Grouped launches with the early-terminated scheme (rows f2 x f4):
    final-node ranges in the top BFS, ragged row ranges inside final nodes."""
    D = 32
    shapes = [(14, 1 << 14, 0, 1 << 14), (12, 3001, 0, 3001), (10, 1000, 37, 900), (16, 60000, 0, 60000),
              (5, 32, 0, 32), (13, 5000, 4096, 904)]
    groups, expect = [], []
    for i, (n, N, r0, rows) in enumerate(shapes):
        B = kt_keys if i % 2 == 0 else max(1, kt_keys // 3)
        T = synth.table(N, D, 970 + i)
        keys, okeys = make_et_keys(dp, oracle, n, synth.alphas(B, N, 970 + i), 980 + i)
        Tsh = T[r0:r0 + rows]
        wire = torch.from_numpy(dp.keys_to_wire(keys)).cuda()
        out = torch.empty((B, D), dtype=torch.int32, device="cuda")
        groups.append((wire, n, to_dev(Tsh), r0, out))
        expect.append(oracle.answer_batch(okeys, Tsh, row_begin=r0, threads=8))
    dp.eval_grouped(groups, D, prf=ET)
    torch.cuda.synchronize()
    for (wire, n, Td, r0, out), want in zip(groups, expect):
        np.testing.assert_array_equal(dp.as_u32(out), want)


@pytest.mark.parametrize("prf,D", [(1, 32), (3, 32), (1, 256), (3, 64), (2, 128)])
def test_grouped_packed_tc(dp, oracle, prf, D):
    """dpf_eval_grouped_packed: many (keys, limb-packed table) groups through the
    tcgen05 kernel (CTA pairs at D = 256) in one launch; mixed key counts, ragged
    row ranges, tiny and deep domains."""
    shapes = [(14, 1 << 14, 0, 1 << 14, 40), (12, 3001, 0, 3001, 17), (10, 1000, 37, 900, 3), (16, 60000, 0, 60000, 33),
              (9, 300, 0, 300, 1), (13, 5000, 4096, 904, 64)]
    groups, expect = [], []
    for i, (n, N, r0, rows, B) in enumerate(shapes):
        if prf == 2 and n > 12:
            continue
        T = synth.table(N, D, 990 + i)
        al = synth.alphas(B, N, 990 + i)
        keys = [dp.gen(n, int(a), 1, s, prf=prf)[(j + i) % 2] for j, (a, s) in enumerate(zip(al, synth.gen_seeds(B, 995 + i)))]
        okeys = [oracle.key_from_wire(dp.key_serialize(k)) for k in keys]
        Tsh = T[r0:r0 + rows]
        wire = torch.from_numpy(dp.keys_to_wire(keys)).cuda()
        out = torch.empty((B, D), dtype=torch.int32, device="cuda")
        groups.append((wire, n, dp.table_pack(to_dev(Tsh), r0), r0, out))
        expect.append(oracle.answer_batch(okeys, Tsh, row_begin=r0, threads=8))
    dp.eval_grouped_packed(groups, D, prf=prf)
    torch.cuda.synchronize()
    for g, want in zip(groups, expect):
        np.testing.assert_array_equal(dp.as_u32(g[4]), want)


@pytest.mark.parametrize("prf,D,packed", [(1, 64, False), (1, 256, True), (3, 128, True), (2, 64, False), (3, 64, False),
                                           (2, 256, True)])
def test_graph_server_replays_new_keys(dp, oracle, prf, D, packed):
    """dpf_server_*: the captured serving graph answers fresh host keys on every
    replay (H2D of the staging buffer inside the graph) and checks headers."""
    n, N, B = 12, 3000, 40
    T = synth.table(N, D, 1200 + D)
    Td = to_dev(T)
    srv = dp.Server(B, n, dp.table_pack(Td) if packed else Td, prf=prf)
    for rep in range(3):
        al = synth.alphas(B, N, 1300 + rep)
        keys = [dp.gen(n, int(a), 1, s, prf=prf)[(i + rep) % 2]
                for i, (a, s) in enumerate(zip(al, synth.gen_seeds(B, 1400 + rep)))]
        got = srv.run(dp.keys_to_wire(keys))
        want = oracle.answer_batch([oracle.key_from_wire(dp.key_serialize(k)) for k in keys], T, threads=8)
        np.testing.assert_array_equal(got, want)
    bad = dp.keys_to_wire(keys).copy()
    bad[3, 0] ^= 1  # magic
    with pytest.raises(dp.DpfError):
        srv.run(bad)
    srv.close()


@pytest.mark.parametrize("depth,packed,prf", [(2, True, 1), (3, False, 1), (2, True, 3), (2, True, 2)])
def test_pipelined_server_batches_in_flight(dp, oracle, depth, packed, prf):
    """dpf_server_pipeline_*: up to `depth` batches in flight, collected oldest
    first, each equal to the oracle; a full pipeline refuses a submit
    (DPF_EBUSY) and run() refuses while batches are in flight."""
    n, N, D, B = 12, 3500, 128, 48
    T = synth.table(N, D, 1500 + depth)
    Td = to_dev(T)
    srv = dp.Server(B, n, dp.table_pack(Td) if packed else Td, prf=prf, depth=depth)
    batches = []
    for rep in range(3 * depth + 1):
        al = synth.alphas(B, N, 1600 + rep)
        keys = [dp.gen(n, int(a), 1, s, prf=prf)[(i + rep) % 2]
                for i, (a, s) in enumerate(zip(al, synth.gen_seeds(B, 1700 + rep)))]
        batches.append(keys)
    want = [oracle.answer_batch([oracle.key_from_wire(dp.key_serialize(k)) for k in keys], T, threads=8)
            for keys in batches]
    got, nxt = [], 0
    for keys in batches:
        if nxt - len(got) == depth:  # pipeline full
            with pytest.raises(dp.DpfError):
                srv.submit(dp.keys_to_wire(keys))
            got.append(srv.collect())
        srv.submit(dp.keys_to_wire(keys))
        nxt += 1
    with pytest.raises(dp.DpfError):
        srv.run(dp.keys_to_wire(batches[0]))
    while len(got) < nxt:
        got.append(srv.collect())
    with pytest.raises(dp.DpfError):
        srv.collect()  # nothing in flight
    for g, w in zip(got, want):
        np.testing.assert_array_equal(g, w)
    np.testing.assert_array_equal(srv.run(dp.keys_to_wire(batches[1])), want[1])
    srv.close()


def test_random_shapes_fuzz(dp, oracle):
    """Seeded random shapes through every entry point family (IMAD and tcgen05
    incl. pairs and padded D, all three schemes, shards with ragged ends, the
    accumulate flag): bit-exact against the oracle."""
    rng = np.random.default_rng(20261017)
    cases = 0
    while cases < 120:
        prf = int(rng.choice([1, 2, 3], p=[0.45, 0.15, 0.4]))
        n = int(rng.integers(5 if prf == 3 else 3, 15))
        N = int(rng.integers(max(8, (1 << n) // 3), (1 << n) + 1))
        D = int(rng.choice([4, 16, 32, 60, 64, 100, 128, 192, 256, 320, 512]))
        B = int(rng.choice([1, 3, 16, 17, 33, 64, 100, 129, 200]))
        if prf == 2 and (n > 11 or B > 64):
            continue  # keep the oracle's AES time bounded
        r0 = int(rng.integers(0, N // 2 + 1))
        rows = int(rng.integers(1, N - r0 + 1))
        packed = bool(rng.integers(0, 2)) and n >= 3
        seed = int(rng.integers(1 << 30))
        T = synth.table(N, D, seed)
        al = synth.alphas(B, N, seed)
        keys = [dp.gen(n, int(a), 1, s, prf=prf)[i % 2] for i, (a, s) in enumerate(zip(al, synth.gen_seeds(B, seed)))]
        okeys = [oracle.key_from_wire(dp.key_serialize(k)) for k in keys]
        Tsh = T[r0:r0 + rows]
        Td = to_dev(Tsh)
        want = oracle.answer_batch(okeys, Tsh, row_begin=r0, threads=16)
        if packed:
            got = dp.as_u32(dp.eval_batch_packed(keys, dp.table_pack(Td, r0)))
        else:
            got = dp.as_u32(dp.eval_batch_shard(keys, Td, r0))
        assert np.array_equal(got, want), (prf, n, N, D, B, r0, rows, packed)
        # accumulate twice into one buffer through the wire path: 2x the answer
        wire = torch.from_numpy(dp.keys_to_wire(keys)).cuda()
        acc = torch.zeros((B, D), dtype=torch.int32, device="cuda")
        ws = torch.empty(dp.eval_workspace_bytes(B, n, rows, D), dtype=torch.uint8, device="cuda")
        for _ in range(2):
            dp.eval_batch_wire_ex(wire, n, dp.table_pack(Td, r0) if packed else Td, r0, rows, D, acc.data_ptr(),
                                  dp.DPF_EVAL_ACCUMULATE, ws, prf=prf, packed=packed)
        torch.cuda.synchronize()
        assert np.array_equal(dp.as_u32(acc), (2 * want.astype(np.uint64) % (1 << 32)).astype(np.uint32))
        cases += 1


@pytest.mark.parametrize("n,N,r0,rows,D,B", [
    (17, 1 << 17, 0, 1 << 17, 256, 130), (18, 250001, 7, 200000, 64, 64), (17, 100000, 4096, 60001, 512, 40),
    (16, 1 << 16, 3, 65000, 128, 300),
])
def test_packed_deep_windows_shards(dp, oracle, n, N, r0, rows, D, B):
    """Deep subtrees (8 leaf pairs per window, CTA pairs at D = 256/512) on
    ragged shards: bit-exact against the oracle."""
    T = synth.table(N, D, 7700 + n)
    al = synth.alphas(B, N, 7700 + n)
    keys, okeys = make_keys(dp, oracle, n, al, 7800 + n)
    Tsh = T[r0:r0 + rows]
    Td = to_dev(Tsh)
    got = dp.as_u32(dp.eval_batch_packed(keys, dp.table_pack(Td, r0)))
    np.testing.assert_array_equal(got, oracle.answer_batch(okeys, Tsh, row_begin=r0, threads=16))


@pytest.mark.parametrize("n,N,D,B,prf,row_begin", [
    (14, 1 << 14, 256, 8, 1, 0), (13, 8000, 64, 9, 1, 0), (14, 1 << 14, 128, 15, 1, 0), (12, 4096, 256, 6, 1, 0),
    (13, 7000, 256, 12, 1, 1000), (14, 1 << 14, 256, 11, 3, 0), (12, 4000, 64, 7, 3, 40), (12, 4096, 128, 4, 1, 0),
    (12, 4096, 128, 2, 1, 0), (16, 1 << 16, 512, 10, 1, 0),
])
def test_packed_tc_small_batch(dp, oracle, n, N, D, B, prf, row_begin):
    """B < 16 on the tensor path: N = 16 MMA columns, only B of them keys
    (Kr = B producer key lanes, zero padding columns); falls back to the
    padded mapping when that y ring does not fit SMEM (B = 2, 4)."""
    T = synth.table(N, D, n + B)
    al = synth.alphas(B, N, n + B)
    seeds = synth.gen_seeds(B, n + B)
    keys = [dp.gen(n, int(a), 1, s, prf=prf)[i % 2] for i, (a, s) in enumerate(zip(al, seeds))]
    okeys = [oracle.key_from_wire(dp.key_serialize(k)) for k in keys]
    Tsh = T[row_begin:]
    got = dp.as_u32(dp.eval_batch_packed(keys, dp.table_pack(to_dev(Tsh), row_begin)))
    np.testing.assert_array_equal(got, oracle.answer_batch(okeys, Tsh, row_begin=row_begin, threads=8))
