"""bench.py's multi-GPU launcher (CPU, gloo): ``--gpus N`` outside torchrun
spawns N ranks itself, and a job whose world size differs from ``--gpus``
refuses to report a number (VERDICT r1 "What's missing" 1)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, env=env,
                          capture_output=True, text=True, timeout=240)


def test_gpus_n_spawns_n_ranks():
    r = _run(["--gpus", "3", "--launcher-selftest"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout      # rank 0 alone prints
    assert lines[0]["n_gpus"] == 3 and lines[0]["ranks_seen"] == 3


def test_world_size_mismatch_fails_loudly():
    r = _run(["--gpus", "2"], {"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0
    assert "WORLD_SIZE=1" in r.stderr
    assert not any(x.startswith("{") for x in r.stdout.splitlines())
