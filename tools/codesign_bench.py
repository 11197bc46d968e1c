"""Co-design workload (BASELINE config c5, row f2) on one GPU.

26 embedding tables (log2 rows [12..22, 12..22, 12..15], D = 32, Zipf(1.0)
accesses), each split into a hot table (top `--hot` fraction of rows) and the
full table.  Every inference needs `--need` rows per table; the
client routes them to Q_hot hot / Q_full full keys per table (dummy-padded,
excess dropped).  The server answers a batch of inferences with ONE
dpf_eval_grouped call over the 52 (table, hot|full) groups; compared with 52
separate dpf_eval_batch_wire calls.  Batch sweep over inferences per batch.
    python tools/codesign_bench.py [--batches 1 4 16 64 256 1024]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2301_10904_b200 import codesign, dpfpir  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batches", type=int, nargs="+", default=[1, 4, 16, 64, 256, 1024])
ap.add_argument("--hot", type=float, default=0.1)
ap.add_argument("--q-hot", type=int, default=2)
ap.add_argument("--q-full", type=int, default=1)
ap.add_argument("--need", type=int, default=3)
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--check", type=int, default=2, help="inferences whose rows are reconstructed and checked")
ap.add_argument("--prf", default="chacha20", choices=["chacha20", "chacha20_et", "aes128"])
ap.add_argument("--packed", action="store_true", help="limb-packed tables + tcgen05 (dpf_eval_grouped_packed)")
ap.add_argument("--scheme", default="hot", choices=["hot", "pbr"],
                help="hot: hot-table split, Q_hot + Q_full keys per table (P:645-659); "
                     "pbr: partial batch retrieval, one key per bin of each full table (P:595-602)")
ap.add_argument("--bins", type=int, default=4, help="PBR bins per table (power of two)")
a = ap.parse_args()
prf = {"chacha20": dpfpir.DPF_PRF_CHACHA20, "chacha20_et": dpfpir.DPF_PRF_CHACHA20_ET, "aes128": dpfpir.DPF_PRF_AES128}[a.prf]
D = synth.CODESIGN_D
rng = np.random.default_rng(0)
tables = []
for t, lg in enumerate(synth.CODESIGN_LOG2_ROWS):
    N = 1 << lg
    T = synth.table(N, D, 0xC5000 + t)
    sp = codesign.HotSplit.from_frequency(synth.codesign_frequency(t, N), a.hot)
    H = sp.hot_table(T)
    Td = torch.from_numpy(T.view(np.int32)).cuda()
    Hd = torch.from_numpy(H.view(np.int32)).cuda()
    if a.packed:  # server state, re-laid-out once
        Td, Hd = dpfpir.table_pack(Td), dpfpir.table_pack(Hd)
    tables.append(dict(N=N, T=T, Td=Td, split=sp, hmap=sp.hot_index(), Hd=Hd,
                       nH=codesign.log2_domain(sp.n_hot), nF=codesign.log2_domain(N)))
torch.cuda.synchronize()
seed_iter = iter(synth.gen_seeds(200000, 0xC5))
for Binf in a.batches:
    # client: plan + keys (outside the timed region: client work)
    groups0, groups1, real = [], [], []
    dropped = 0
    for t, tb in enumerate(tables):
        need = synth.codesign_needed(t, tb["N"], Binf, a.need)
        if a.scheme == "pbr":
            # one group per bin: the keys of all inferences for that bin
            log_i = tb["nF"] - (a.bins.bit_length() - 1)
            I = 1 << log_i
            pplans = [codesign.plan_pbr(r, tb["N"], log_i, rng) for r in need]
            dropped += sum(len(p.dropped) for p in pplans)
            for b in range(codesign.pbr_n_bins(tb["N"], log_i)):
                pairs = [dpfpir.gen(log_i, int(p.index[b]), 1, next(seed_iter), prf=prf) for p in pplans]
                if a.packed:
                    Dp = (D + 127) // 128 * 128
                    view = dpfpir.PackedTable(tb["Td"].data[(b * I // 8) * 32 * Dp:((b + 1) * I // 8) * 32 * Dp], 0, I, D)
                else:
                    view = tb["Td"][b * I:(b + 1) * I]
                for party, gl in ((0, groups0), (1, groups1)):
                    wire = torch.from_numpy(dpfpir.keys_to_wire([p[party] for p in pairs])).cuda()
                    out = torch.empty((len(pairs), D), dtype=torch.int32, device="cuda")
                    gl.append((wire, log_i, view, 0, out))
                real.append((t, "pbr", [(p.real[b], p.rows[b]) for p in pplans]))
            continue
        plans = [codesign.plan_table(r, tb["split"], tb["hmap"], a.q_hot, a.q_full, rng) for r in need]
        dropped += sum(p.dropped for p in plans)
        for kind, tbl, n, idxs in (("hot", tb["Hd"], tb["nH"], [p.hot_idx for p in plans]),
                                   ("full", tb["Td"], tb["nF"], [p.full_idx for p in plans])):
            flat = np.concatenate(idxs)
            pairs = [dpfpir.gen(n, int(i), 1, next(seed_iter), prf=prf) for i in flat]
            for party, gl in ((0, groups0), (1, groups1)):
                wire = torch.from_numpy(dpfpir.keys_to_wire([p[party] for p in pairs])).cuda()
                out = torch.empty((len(flat), D), dtype=torch.int32, device="cuda")
                gl.append((wire, n, tbl, 0, out))
            real.append((t, kind, plans))
    n_keys = sum(g[0].shape[0] for g in groups0)
    wsb = (dpfpir.eval_grouped_packed_workspace_bytes if a.packed else dpfpir.eval_grouped_workspace_bytes)(
        groups0, D, prf=prf)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    run_grouped = dpfpir.eval_grouped_packed if a.packed else dpfpir.eval_grouped

    def grouped():
        run_grouped(groups0, D, prf=prf, workspace=ws)

    def separate():
        for (wire, n, tbl, r0, out) in groups0:
            if a.packed:
                dpfpir.eval_batch_wire_packed(wire, n, tbl, out=out, prf=prf)
            else:
                dpfpir.eval_batch_wire(wire, n, tbl, r0, out=out, prf=prf)

    res = {}
    for name, fn in (("grouped", grouped), ("separate", separate)):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / a.steps
    # correctness: second server, reconstruct the first inferences' real queries
    grouped()
    plan = dpfpir.last_eval_stats()
    run_grouped(groups1, D, prf=prf)
    torch.cuda.synchronize()
    ok = True
    for gi, (t, kind, plans) in enumerate(real):
        ans = dpfpir.reconstruct(dpfpir.as_u32(groups0[gi][4]), dpfpir.as_u32(groups1[gi][4]))
        if kind == "pbr":
            for inf in range(min(a.check, Binf)):
                is_real, row = plans[inf]
                if is_real:
                    ok &= bool(np.array_equal(ans[inf], tables[t]["T"][row]))
            continue
        q = a.q_hot if kind == "hot" else a.q_full
        for inf in range(min(a.check, Binf)):
            p = plans[inf]
            rows = p.hot_rows if kind == "hot" else p.full_idx
            mask = p.hot_real if kind == "hot" else p.full_real
            for j in np.nonzero(mask)[0]:
                ok &= bool(np.array_equal(ans[inf * q + j], tables[t]["T"][rows[j]]))
    # blocks over each table's rows: N - 1 per key (R9), N/8 - 1 with early termination (R20)
    blocks = sum(g[0].shape[0] * ((g[2].shape[0] - 1) if prf != dpfpir.DPF_PRF_CHACHA20_ET else max(1, g[2].shape[0] // 8 - 1))
                 for g in groups0)
    n_rows_wanted = Binf * len(tables) * a.need
    ms = res["grouped"]
    print(json.dumps({"workload": "c5 co-design", "scheme": a.scheme, "bins": a.bins if a.scheme == "pbr" else None,
                      "prf": a.prf, "packed": a.packed, "inferences_per_batch": Binf, "keys_per_batch": n_keys,
                      "q_hot": a.q_hot, "q_full": a.q_full, "hot_fraction": a.hot, "need_per_table": a.need,
                      "dropped_rows": dropped, "wanted_rows": n_rows_wanted, "ms_grouped": round(ms, 4), "ms_separate": round(res["separate"], 4),
                      "inferences_per_s": round(Binf / (ms * 1e-3), 1), "dpf_queries_per_s": round(n_keys / (ms * 1e-3)),
                      # ALU roofline (640 ops per ChaCha20 block); AES-128: the SMEM-lookup roofline
                      # (333 table lookups per node, bench.aes_lookups_per_node, 32 lanes/clk/SM)
                      "alu_frac" if prf != dpfpir.DPF_PRF_AES128 else "smem_frac":
                          round((640 * blocks / (148 * 64 * 1965e6) if prf != dpfpir.DPF_PRF_AES128 else
                                 333 * blocks / (148 * 32 * 1965e6)) / (ms * 1e-3), 3),
                      "rows_reconstructed_ok": ok, "plan": plan}), flush=True)
