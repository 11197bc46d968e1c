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
