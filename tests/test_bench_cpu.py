"""bench.py's contract pieces that run without a GPU: the reference arm's
JSON line (CPU only), and rank > 0 of the reference arm exiting quietly."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                          capture_output=True, text=True, env=e, timeout=300)


def test_reference_arm_json(ref):
    p = run(["--impl", "reference", "--steps", "3", "--warmup", "3", "--cpu-sample", "20000"])
    assert p.returncode == 0, p.stderr
    lines = [l for l in p.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"].startswith("3D Euler flux Gpoints/s")
    assert d["unit"] == "Gpoints/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 3 and d["warmup"] == 3
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_other_ranks_exit_zero(ref):
    p = run(["--impl", "reference", "--steps", "3", "--warmup", "3", "--cpu-sample", "1000"],
            env={"RANK": "1", "WORLD_SIZE": "2"})
    assert p.returncode == 0 and p.stdout.strip() == ""


def test_warmup_floor():
    p = run(["--warmup", "2"])
    assert p.returncode != 0


@pytest.mark.parametrize("config", ["cons2prim1d", "jacobian3d", "axpy", "vmag2"])
def test_reference_arm_other_configs(ref, config):
    p = run(["--impl", "reference", "--config", config, "--steps", "3", "--warmup", "3",
             "--cpu-sample", "5000", "--n", "5000"])
    assert p.returncode == 0, p.stderr
    assert json.loads(p.stdout)["config"]["config"] == config
