"""bench.py's multi-rank launcher on CPU (no GPU): `--gpus N` without
torchrun starts N ranks itself, they rendezvous on 127.0.0.1 (gloo here),
broadcast packed words, deal every tile exactly once through the C ABI and
reduce their timings max-over-ranks; rank 0 alone prints one JSON line with
n_gpus = N.  Under torchrun, WORLD_SIZE must equal --gpus."""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _run(args, env=None, timeout=300):
    e = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    if env:
        e.update(env)
    return subprocess.run([sys.executable, str(ROOT / "bench.py")] + args, capture_output=True, text=True,
                          timeout=timeout, env=e, cwd=str(ROOT))


@pytest.mark.parametrize("n", [2, 4])
def test_bench_spawns_ranks_without_torchrun(n):
    r = _run(["--gpus", str(n), "--plumbing-check"])
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["world_size"] == n
    assert d["tiles_dealt"] == d["tiles_total"] and d["broadcast_ok"]


def test_bench_rejects_world_size_mismatch():
    r = _run(["--gpus", "2", "--plumbing-check"], env={"WORLD_SIZE": "3", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2 and "WORLD_SIZE=3" in r.stderr
