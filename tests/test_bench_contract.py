"""bench.py's driver contract on CPU: the reference arm (`--impl reference`,
the oracle on the host cores) prints ONE JSON line with the required keys, and
under torchrun-style env (RANK != 0) a non-zero rank exits 0 without output.
The GPU arm needs a B200 (bench.py refuses to run without CUDA: no CPU
fallback), which is also checked here."""
import json
import os
import subprocess
import sys

import pytest
from conftest import ROOT

REQUIRED = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"}


def _run(args, env_extra=None):
    env = dict(os.environ)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=600, env=env, cwd=ROOT)


def test_reference_arm_json_line():
    r = _run(["--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "3"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert REQUIRED <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["N"] == 1024 and d["config"]["D"] == 16


def test_reference_arm_nonzero_rank_is_silent():
    r = _run(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "3"],
             {"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_gpu_arm_refuses_without_cuda():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    r = _run(["--config", "c1", "--steps", "1", "--warmup", "3"])
    assert r.returncode != 0
    assert "CUDA" in (r.stdout + r.stderr)


def test_reference_arm_is_pure_oracle_and_same_config():
    """The reference arm never loads libdpfpir (keys from the oracle's Gen) and
    its config dict is the GPU arm's (bench.workload_config)."""
    r = _run(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "3", "--gpus", "2"])
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    import bench
    assert d["config"] == bench.workload_config(bench.synth.CONFIGS["c1"], "chacha20", 2)
    assert d["n_gpus"] == 2 and "cpu" in d["cpu_baseline"]
    src = open(os.path.join(ROOT, "bench.py")).read()
    ref = src[src.index("def run_reference"):src.index("# ---------------------------------------------------------------------- our arm")]
    assert "dpfpir" not in ref and "paper_2301_10904_b200" not in ref


def test_gpus_n_self_spawns_n_ranks():
    """`bench.py --gpus 2` without WORLD_SIZE re-launches itself under
    torch.distributed.run with 2 ranks (the GPU arm is replaced by --dry-env,
    which prints each rank's launch environment)."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-env"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    rows = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert sorted(x["rank"] for x in rows) == [0, 1]
    assert all(x["world"] == 2 and x["master_addr"] == "127.0.0.1" for x in rows)
    assert sorted(x["local_rank"] for x in rows) == [0, 1]


def test_world_size_must_match_gpus():
    r = _run(["--gpus", "4", "--dry-env"], {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and "WORLD_SIZE=2" in (r.stdout + r.stderr)


def test_gpus_1_runs_in_process():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--dry-env"], capture_output=True,
                       text=True, timeout=120, env=env, cwd=ROOT)
    assert r.returncode == 0
    rows = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert rows == [{"rank": 0, "world": 1, "local_rank": 0, "master_addr": None}]


def test_parity_miss_suppresses_line_and_fails(capsys):
    import bench
    line = {"metric": bench.METRIC, "value": 1.0}
    assert bench.emit(line, {"reconstruct_all_queries": True, "bit_exact_vs_oracle": False}) == 3
    out = capsys.readouterr()
    assert out.out == "" and "PARITY FAILURE" in out.err
    assert bench.emit(line, {}) == 3  # no checks ran: also a failure
    capsys.readouterr()
    assert bench.emit(line, {"reconstruct_all_queries": True, "oracle_sample_keys": 4,
                             "bit_exact_vs_oracle": True}) == 0
    assert json.loads(capsys.readouterr().out)["value"] == 1.0


def test_aes_circuit_count():
    """gates of BMP13 S-box (113), Maximov MixColumns (92),
    AddRoundKey, key expansion (+ Rcon bits), / 32 bit-slices per word."""
    import bench
    gates = 10 * 32 * 113 + 9 * 8 * 92 + 11 * 256 + 10 * (4 * 113 + 128) + 16
    assert bench.aes_alu_ops_per_node() == gates / 32


def test_aes_lookup_count():
    """distinct S-box inputs of one tree node, counted over the
    byte positions from which state bytes the two blocks' states can differ:
    round 1 (key XOR 0^120||c): byte 15 only; round 2: the bytes that round 1
    computed from byte 15 -- ShiftRows moves byte 15 (row 3, column 3) to
    column 0 and MixColumns spreads it over column 0's 4 bytes; round >= 3:
    every byte.  A lookup per (round, distinct input) plus 4 per key-schedule
    round."""
    import bench
    diff = {15}  # state bytes (index r + 4c) that differ between the two blocks
    n = 0
    for rnd in range(1, 11):
        n += 16 + len(diff) + 4
        # next round's differing bytes: ShiftRows new (r, c) = old (r, c + r); MixColumns mixes a column
        moved = {r + 4 * ((c - r) % 4) for r, c in ((i % 4, i // 4) for i in diff)}
        diff = {r + 4 * c for c in {i // 4 for i in moved} for r in range(4)}
    assert n == bench.AES_LOOKUPS_PER_NODE == 333


def test_roofline_of_runs_on_cpu_with_plan_stats():
    """roofline_of (the bench line's roofline object) from host-only plan
    stats: it runs without a GPU, names the timed kernel instantiation, and
    drops the committed ncu traffic when that capture is of another kernel."""
    import argparse
    import bench
    import synth
    from paper_2301_10904_b200 import dpfpir
    w = synth.CONFIGS["c3"]
    stats = dpfpir.eval_plan(w.B, w.log_n, w.N, w.D, packed=True)
    args = argparse.Namespace(prf="chacha20", config="c3")
    r = bench.roofline_of(args, w, w.N, 0, 1, stats, [10.0], 10.1, 25000.0, True)
    assert r["bound"] == "alu" and 0.8 < r["frac"] < 1.0
    assert r["timed_kernel"] == dpfpir.kernel_name(stats["kernel_id"])
    assert r["timed_kernel"].startswith("fused_eval_tc_kernel<PrfChacha, 16, ")
    if r["traffic_kernel"] != r["timed_kernel"]:
        assert r["traffic"] is None
    stats["kernel_id"] ^= 2  # claim the other CTA-pair variant: the capture no longer applies
    r2 = bench.roofline_of(args, w, w.N, 0, 1, stats, [10.0], 10.1, 25000.0, True)
    assert r2["traffic"] is None
