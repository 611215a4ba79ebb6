"""bench.py's multi-rank plumbing on CPU: ``--gpus 2`` outside torchrun
re-executes itself under torch.distributed.run (gloo here, ``--selftest``),
shards the config-3 batch contiguously, takes the max over ranks and prints one
line from rank 0 whose result checksum equals the single-rank run."""

from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, env=None):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=600, env={**os.environ, **(env or {})})
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    return r, lines


def test_bench_spawns_ranks_and_shards_config3():
    r1, l1 = _run("--gpus", "1", "--selftest", "--steps", "1", "--warmup", "0")
    assert r1.returncode == 0, r1.stderr[-2000:]
    r2, l2 = _run("--gpus", "2", "--selftest", "--steps", "1", "--warmup", "0")
    assert r2.returncode == 0, r2.stderr[-2000:]
    assert len(l1) == 1 and len(l2) == 1  # rank 0 alone prints
    a, b = json.loads(l1[0]), json.loads(l2[0])
    assert a["n_gpus"] == 1 and b["n_gpus"] == 2
    assert b["shards"] == [[0, 4], [4, 8]]
    assert a["checksum"] == b["checksum"]
    assert b["value"] > 0


def test_bench_rejects_world_size_mismatch():
    r, _ = _run("--gpus", "2", "--selftest", env={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2 and "WORLD_SIZE" in r.stderr
