"""bench.py --impl reference runs on the host only (no GPU): the oracle on the
same workload as our arm's line for that N -- C3 at N = 1, the whole C4 array
at N > 1 (rank 0 only; other ranks exit quietly) -- with the contract's keys."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(world, rank, n_total):
    env = dict(os.environ, WORLD_SIZE=str(world), RANK=str(rank))
    cmd = [sys.executable, "bench.py", "--impl", "reference", "--gpus", str(world), "--steps", "2",
           "--warmup", "1", "--n-total", str(n_total)]
    return subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)


@pytest.mark.parametrize("world", [1, 2])
def test_reference_arm_line(world):
    sys.path.insert(0, ROOT)
    import bench

    n = (1 << 20) + 3
    r = _run(world, 0, n)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == world and d["steps"] == 2
    assert d["config"]["n_total"] == n
    assert d["config"]["workload"] == bench.c3c4_workload(world, n, "f16", False)
    assert d["scaling"] == ("strong" if world > 1 else "weak")
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] == d["value"] > 0 and cb["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_print_nothing():
    r = _run(2, 1, 1 << 16)
    assert r.returncode == 0 and not [l for l in r.stdout.splitlines() if l.startswith("{")]
