"""GPU parity of partial batch retrieval (dpf_eval_pbr, row f2; P:595-602,
reading R21): the device answers of every bin equal the oracle's pbr_answer
bit-exactly, on row-major (IMAD) and limb-packed (tcgen05) tables, ChaCha20,
early termination and AES-128, with ragged last bins; the client planner's
kept rows reconstruct to the table rows."""
import numpy as np
import pytest

import synth
from paper_2301_10904_b200 import codesign

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


def _case(dp, oracle, N, log_i, D, B, seed, packed=False, prf=None, check_clients=None):
    prf = dp.DPF_PRF_CHACHA20 if prf is None else prf
    T = synth.table(N, D, seed)
    Td = torch.from_numpy(T.view(np.int32)).cuda()
    table = dp.table_pack(Td) if packed else Td
    nb = codesign.pbr_n_bins(N, log_i)
    rng = np.random.default_rng(seed)
    plans = [codesign.plan_pbr(rng.integers(0, N, size=nb + 2), N, log_i, rng) for _ in range(B)]
    seeds = iter(synth.gen_seeds(2 * nb * B, seed))
    pairs = [[dp.gen(log_i, int(plans[c].index[b]), 1, next(seeds), prf=prf) for c in range(B)] for b in range(nb)]
    got = []
    for party in (0, 1):
        keys = [pairs[b][c][party] for b in range(nb) for c in range(B)]  # bin-major
        wire = torch.from_numpy(dp.keys_to_wire(keys)).cuda()
        got.append(dp.as_u32(dp.eval_pbr(wire, B, log_i, table, prf=prf)).reshape(nb, B, D))
    torch.cuda.synchronize()
    clients = range(B) if check_clients is None else check_clients
    for party in (0, 1):
        okeys = [[oracle.key_from_wire(dp.key_serialize(pairs[b][c][party])) for c in clients] for b in range(nb)]
        want = oracle.pbr_answer(okeys, T, log_i, threads=8)
        np.testing.assert_array_equal(got[party][:, list(clients)], want)
    rec = (got[0].astype(np.uint64) + got[1]) & 0xFFFFFFFF
    for c in range(B):
        p = plans[c]
        for b in np.nonzero(p.real)[0]:
            np.testing.assert_array_equal(rec[b, c], T[p.rows[b]])


def test_pbr_rowmajor_chacha(dp, oracle):
    _case(dp, oracle, 1 << 12, 8, 32, 5, 11)


def test_pbr_rowmajor_ragged_last_bin(dp, oracle):
    _case(dp, oracle, 3000, 9, 16, 3, 12)          # 6 bins, the last one 440 rows


def test_pbr_packed_tcgen05(dp, oracle):
    _case(dp, oracle, 1 << 14, 10, 128, 20, 13, packed=True)


def test_pbr_packed_ragged_et(dp, oracle):
    _case(dp, oracle, 5000, 8, 64, 17, 14, packed=True, prf=dp.DPF_PRF_CHACHA20_ET)


def test_pbr_rowmajor_aes(dp, oracle):
    _case(dp, oracle, 1 << 10, 7, 8, 2, 15, prf=dp.DPF_PRF_AES128)


def test_pbr_c5_table_size(dp, oracle):
    """The largest c5 table (2^22 rows x D = 32) in 16 bins, 64 clients; the
    oracle checks 3 of them, reconstruction checks all."""
    _case(dp, oracle, 1 << 22, 18, 32, 64, 16, packed=True, check_clients=[0, 31, 63])


def test_pbr_rejects_bad_shapes(dp):
    T = torch.zeros((1024, 8), dtype=torch.int32, device="cuda")
    wire = torch.zeros((3, dp.key_wire_size(5)), dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):
        dp.eval_pbr(wire, 1, 5, T)  # 32 bins need 32 keys
    assert dp.eval_pbr_workspace_bytes(1, 2, 1024, 8, packed=True) == 0  # packed bins need I >= 8
