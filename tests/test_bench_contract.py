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
