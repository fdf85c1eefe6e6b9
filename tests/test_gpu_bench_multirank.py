"""The bench's N > 1 code path (sharding, allreduce of the fp64 partial /
exact limbs, max-over-ranks timing, rank-0 JSON) under torchrun with two
ranks on the single GPU of the test box (gloo, TCR_BENCH_SHARED_GPU=1 --
a code-path test, not a measurement)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["default", "exact"])
def test_bench_two_ranks_shared_gpu(algo):
    env = dict(os.environ, TCR_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3", "--e2e-steps", "1",
           "--n-per-rank", str(1 << 24), "--algo", algo]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 prints exactly one JSON line
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["n_total"] == 2 << 24
    assert d["gpu_launches"] >= 3 and d["e2e"]["h2d_bytes_per_step"] == 2 << 24
    assert d["test_mode"].startswith("shared-gpu")


@pytest.mark.gpu
def test_bench_c4_strong_two_ranks_shared_gpu():
    """C4 as BASELINE.json defines it: a fixed global n = 2^33 cut over the
    ranks (strong scaling), the timed result checked against the exact
    oracle of the whole array (per-rank shard oracles, exact limb
    allreduce), a cpu_baseline for the whole job, and T_1 (rank 0 reducing
    all 2^33 elements alone)."""
    env = dict(os.environ, TCR_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3", "--e2e-steps", "1"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["n_total"] == 1 << 33 and d["config"]["n_per_rank"] == 1 << 32
    assert d["config"]["workload"].startswith("c4")
    ck = d["check"]
    assert ck["within_2^-20_sum_abs"] is True and ck["exact_f64"] != 0.0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] > 0 and cb["cores"] >= 2
    assert d["t1"]["n"] == 1 << 33 and d["t1"]["ms_per_step"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("extra", [[], ["--impl", "reference"], ["--workload", "c5"]])
def test_bench_json_contract_single_gpu(extra):
    """bench.py at N = 1: one JSON line carrying every key of the contract."""
    cmd = [sys.executable, "bench.py", "--steps", "5", "--warmup", "3", "--e2e-steps", "1",
           "--n-total", str(1 << 24), "--cpu-seconds", "1"] + extra
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "cpu_baseline"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3
    assert d["higher_is_better"] is True and d["value"] > 0
    assert "workload" in d["config"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]
    assert cb["cpu_model"] and cb["host_ram_gib"] > 0
    if extra[:2] == ["--impl", "reference"]:
        assert d["config"]["n_total"] == 1 << 24  # the same workload as our arm's line
        assert d["impl"] == "reference"
        assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
        return
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert d["gpu_launches"] == 5  # one launch of the reduction kernel per step
    ck = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(ck)
    if "c5" not in extra:
        assert d["check"]["within_2^-20_sum_abs"] is True  # the timed result vs the oracle
        assert cb["one_thread"]["value"] > 0 and cb["d2h_ms"] > 0
        e = d["e2e"]
        assert e["value"] > 0 and e["h2d_bytes_per_step"] == 2 << 24 and e["d2h_bytes_per_step"] == 4


@pytest.mark.gpu
def test_bench_c5_two_ranks_shared_gpu():
    """C5 at N = 2: whole segments sharded by element count, no collective,
    strong scaling; job element count = the whole C5 workload."""
    env = dict(os.environ, TCR_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--workload", "c5"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    import tcr_inputs as gen

    total = int(gen.offsets_from_lengths(gen.loguniform_lengths(gen.SEED_C5, 1 << 20))[-1])
    assert d["scaling"] == "strong" and d["config"]["n_total"] == total and d["n_gpus"] == 2
    assert d["gpu_launches"] == 3
