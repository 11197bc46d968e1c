"""bench.py on the GPU: the line carries the contract keys and a parity miss
(forced with the DPF_BENCH_INJECT_MISMATCH test hook, which flips one answer
word before the checks) exits non-zero without printing a result line."""
import json
import os
import subprocess
import sys

import pytest
from conftest import ROOT

pytestmark = pytest.mark.gpu


def _bench(args, env_extra=None):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=900, env=env, cwd=ROOT)


def test_bench_c1_line_and_parity():
    r = _bench(["--config", "c1", "--steps", "5", "--warmup", "3"])
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["parity"]["reconstruct_all_queries"] and d["parity"]["bit_exact_vs_oracle"]
    assert d["parity"]["e2e_equals_device_path"]
    assert {"p10", "p50", "p90"} <= set(d["latency_ms"])
    assert d["cpu_baseline"]["single_thread_value"] > 0 and d["cpu_baseline"]["cpu"]
    assert d["roofline"]["bound"] in ("alu", "tensor", "hbm")


@pytest.mark.parametrize("config", ["c1", "c2"])
def test_bench_parity_miss_exits_nonzero(config):
    r = _bench(["--config", config, "--steps", "3", "--warmup", "3", "--no-cpu-baseline"],
               {"DPF_BENCH_INJECT_MISMATCH": "1"})
    assert r.returncode == 3, (r.returncode, r.stderr[-3000:])
    assert r.stdout.strip() == ""
    assert "PARITY FAILURE" in r.stderr


@pytest.mark.parametrize("gpus,config,reduce", [(2, "c2", "nccl"), (3, "c1", "nccl"), (2, "c2", "p2p")])
def test_bench_multi_rank_path_on_one_gpu(gpus, config, reduce):
    """`bench.py --gpus N` end to end (self-launch under torch.distributed.run,
    row shards, the reduce, N > 1 oracle parity on the reduced answers, the
    int32-wrap case, max-over-ranks timing, one line from rank 0) with every
    rank on this box's one GPU (DPF_BENCH_SHARED_GPU: gloo group, host-side
    collectives; --reduce p2p maps rank 0's answers into the other ranks with
    CUDA IPC on the same device).  The driver's multi-GPU run takes the same
    path with NCCL over NVLink."""
    r = _bench(["--gpus", str(gpus), "--config", config, "--steps", "3", "--warmup", "3", "--no-cpu-baseline",
                "--reduce", reduce], {"DPF_BENCH_SHARED_GPU": "1"})
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == gpus and "test_mode" in d
    p = d["parity"]
    assert p["reconstruct_all_queries"] and p["bit_exact_vs_oracle"] and p["e2e_equals_device_path"]
    assert p["wrap_reduce_exact"] and p["wrap_case_exercised"]


def test_bench_multi_rank_parity_miss_exits_nonzero():
    r = _bench(["--gpus", "2", "--config", "c1", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"],
               {"DPF_BENCH_SHARED_GPU": "1", "DPF_BENCH_INJECT_MISMATCH": "1"})
    assert r.returncode != 0, (r.returncode, r.stderr[-3000:])  # every rank exits 3; torchrun reports failure
    assert not [x for x in r.stdout.splitlines() if x.startswith("{")]
