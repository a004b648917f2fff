"""bench.py contract checks that run without a GPU: the reference arm (the oracle on the
host cores) prints one JSON line with the fields the driver reads."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("workload", ["cfg5", "cfg2"])
def test_reference_arm_json_line(workload):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--workload", workload, "--steps", "2", "--warmup", "1",
                          "--cpu-seconds", "0.5"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 1
    assert d["metric"].startswith("energy points/sec") and d["unit"] == "energy points/s"
    assert d["higher_is_better"] is True and d["dtype"] == "f64" and d["vs_baseline"] is None
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert "workload" in d["config"]


def test_reference_arm_nonzero_rank_is_silent():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True,
                         timeout=300, cwd=ROOT, env=env)
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_gpus_n_without_launcher_spawns_ranks_reference_arm():
    """`bench.py --gpus 2` with WORLD_SIZE unset starts its own 2 ranks (torch.distributed.run
    on 127.0.0.1); for the reference arm rank 0 alone runs and prints one line, n_gpus 2."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--workload", "cfg1", "--steps", "2", "--warmup", "1",
                          "--cpu-seconds", "0.3"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0


def test_gpus_n_without_launcher_spawns_ranks_our_arm_fails_loudly_without_gpu():
    """Our arm under the self-launch: both ranks start (gloo process group), and with no
    GPU in this container they fail loudly (no CPU fallback, no JSON line)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present: the launch would run the real benchmark")
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--backend", "gloo", "--workload", "cfg1", "--steps", "1",
                          "--warmup", "1"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT, env=env)
    assert out.returncode != 0
    assert not [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    err = out.stderr
    # torch.distributed.run reports the failed local ranks
    assert "local_rank" in err or "rank" in err.lower(), err[-2000:]
