"""bench.py's multi-rank launcher and its reference-arm contract (CPU; gloo stands in for NCCL)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]


def _run(*argv, env=None, timeout=180):
    e = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    e.update(env or {})
    return subprocess.run([sys.executable, str(REPO / "bench.py"), *argv], capture_output=True, text=True,
                          timeout=timeout, env=e, cwd=REPO)


@pytest.mark.parametrize("n", [2, 3])
def test_gpus_flag_launches_n_ranks(n):
    """`bench.py --gpus N` outside torchrun re-launches itself with N ranks (one process each)."""
    r = _run("--gpus", str(n), "--launch-selftest")
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line == {"n_gpus": n, "ranks": list(range(n)), "local_ranks": list(range(n)), "pids": n}


def test_world_size_mismatch_is_an_error():
    r = _run("--gpus", "4", "--launch-selftest", env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and "WORLD_SIZE=2" in r.stderr


def test_both_arms_share_the_config_dict():
    sys.path.insert(0, str(REPO))
    import bench

    for world in (1, 2, 8):
        cfg = bench.bench_config(world)
        assert cfg["parallelism"] == f"frame-shard x{world} (weak)"
        assert set(cfg) == {"workload", "batch", "h", "w", "window", "levels", "seed_base", "parallelism", "l2"}


def test_host_cores_respects_affinity():
    sys.path.insert(0, str(REPO))
    import bench

    assert 1 <= bench.host_cores() <= len(os.sched_getaffinity(0))
