"""GPU parity at the sizes the bench and DESIGN.md claim:
  * c4 (log_n 24, D 64, B 512) on the LAST of 8 row shards (2^21 rows), in
    bench.py's launch configuration (limb-packed table, tcgen05): >= 4 keys
    against the oracle, and both parties' shard answers reconstruct every
    query (beta T[alpha] inside the shard, 0 outside);
  * the 26-table co-design workload c5 (D = 32, hot/full split, 52 groups) in
    one dpf_eval_grouped launch sequence, every key against the oracle;
  * c3 on the tensor path with 16 keys against the oracle (ChaCha20 and AES-128).
Every comparison is element-wise (assert_array_equal): one wrong word fails."""
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


def to_dev(T):
    return torch.from_numpy(T.view(np.int32)).cuda()


@pytest.mark.parametrize("prf_name", ["chacha20", "chacha20_et"])
def test_c4_last_of_8_shards(dp, oracle, prf_name):
    from paper_2301_10904_b200 import shard
    prf = dp.DPF_PRF_CHACHA20 if prf_name == "chacha20" else dp.DPF_PRF_CHACHA20_ET
    w = synth.CONFIGS["c4"]
    r0, rows = shard.row_range(w.N, 8, 7)
    T = synth.table_rows(w.N, w.D, w.seed, r0, r0 + rows)
    al = synth.alphas(w.B, w.N, w.seed)
    # a quarter of the queries inside this shard so reconstruction sees real rows
    al[: w.B // 4] = r0 + (al[: w.B // 4] % rows)
    pairs = [dp.gen(w.log_n, int(a), 1, s, prf=prf) for a, s in zip(al, synth.gen_seeds(w.B, w.seed))]
    pk = dp.table_pack(to_dev(T), r0)
    wire0 = torch.from_numpy(dp.keys_to_wire([p[0] for p in pairs])).cuda()
    sh0 = dp.as_u32(dp.eval_batch_wire_packed(wire0, w.log_n, pk, prf=prf))
    sh1 = dp.as_u32(dp.eval_batch_packed([p[1] for p in pairs], pk))
    st = dp.last_eval_stats()
    assert st["work_items"] >= 148
    inside = (al >= r0) & (al < r0 + rows)
    want = np.zeros((w.B, w.D), np.uint32)
    want[inside] = T[(al[inside] - r0).astype(np.int64)]
    np.testing.assert_array_equal(dp.reconstruct(sh0, sh1), want)
    sample = [0, 1, 200, w.B - 1]  # two inside, two (almost surely) outside
    ok = [oracle.key_from_wire(dp.key_serialize(pairs[b][0])) for b in sample]
    got = oracle.answer_batch(ok, T, row_begin=r0, threads=4)
    for i, b in enumerate(sample):
        np.testing.assert_array_equal(sh0[b], got[i])


def test_c5_codesign_26_tables(dp, oracle):
    from paper_2301_10904_b200 import codesign
    D = synth.CODESIGN_D
    rng = np.random.default_rng(1)
    n_inf, q_hot, q_full, need = 2, 2, 1, 3
    seeds = iter(synth.gen_seeds(4096, 0xC55))
    groups0, groups1, checks = [], [], []
    for t, lg in enumerate(synth.CODESIGN_LOG2_ROWS):
        N = 1 << lg
        T = synth.table(N, D, 0xC5000 + t)
        sp = codesign.HotSplit.from_frequency(synth.codesign_frequency(t, N), 0.1)
        H = sp.hot_table(T)
        plans = [codesign.plan_table(r, sp, sp.hot_index(), q_hot, q_full, rng)
                 for r in synth.codesign_needed(t, N, n_inf, need)]
        for tbl, n, idx in ((H, codesign.log2_domain(sp.n_hot), np.concatenate([p.hot_idx for p in plans])),
                            (T, codesign.log2_domain(N), np.concatenate([p.full_idx for p in plans]))):
            pairs = [dp.gen(n, int(i), 1, next(seeds)) for i in idx]
            Td = to_dev(tbl)
            for party, gl in ((0, groups0), (1, groups1)):
                wire = torch.from_numpy(dp.keys_to_wire([p[party] for p in pairs])).cuda()
                gl.append((wire, n, Td, 0, torch.empty((len(idx), D), dtype=torch.int32, device="cuda")))
            checks.append((tbl, idx, pairs))
    assert len(groups0) == 52
    dp.eval_grouped(groups0, D)
    dp.eval_grouped(groups1, D)
    torch.cuda.synchronize()
    for gi, (tbl, idx, pairs) in enumerate(checks):
        s0, s1 = dp.as_u32(groups0[gi][4]), dp.as_u32(groups1[gi][4])
        np.testing.assert_array_equal(dp.reconstruct(s0, s1), tbl[idx.astype(np.int64)])
        ok = [oracle.key_from_wire(dp.key_serialize(p[0])) for p in pairs]
        np.testing.assert_array_equal(s0, oracle.answer_batch(ok, tbl, threads=8))


@pytest.mark.parametrize("prf_name", ["chacha20", "aes128"])
def test_c3_tensor_path_16_keys(dp, oracle, prf_name):
    """c3 in bench.py's launch configuration (limb-packed table, CTA pairs, the
    full 256-key batch), 16 keys spread over the batch against the oracle; for
    AES-128 the T-table kernels (64 KB tables beside the rings and a shallower
    DFS stack) at the size the AES bench line claims."""
    prf = {"chacha20": dp.DPF_PRF_CHACHA20, "aes128": dp.DPF_PRF_AES128}[prf_name]
    w = synth.CONFIGS["c3"]
    T = synth.table(w.N, w.D, w.seed)
    al = synth.alphas(w.B, w.N, w.seed)
    pairs = [dp.gen(w.log_n, int(a), 1, s, prf=prf) for a, s in zip(al, synth.gen_seeds(w.B, w.seed))]
    pk = dp.table_pack(to_dev(T))
    wire = torch.from_numpy(dp.keys_to_wire([p[0] for p in pairs])).cuda()
    sh0 = dp.as_u32(dp.eval_batch_wire_packed(wire, w.log_n, pk, prf=prf))
    st = dp.last_eval_stats()
    assert st["keys_per_tile"] == 128  # the bench's CTA-pair configuration
    sample = list(range(0, w.B, 16))
    ok = [oracle.key_from_wire(dp.key_serialize(pairs[b][0])) for b in sample]
    want = oracle.answer_batch(ok, T, threads=16)
    for i, b in enumerate(sample):
        np.testing.assert_array_equal(sh0[b], want[i])
