#!/usr/bin/env python
"""bench.py -- throughput of the MMA-encoded fp16 sum reduction on B200.

Metric (BASELINE.json): reduction throughput in Gelem/s (and HBM GB/s as a
fraction of roofline) at 1/2/4/8 B200.  One step = one pass of the whole hot
path (tcr_reduce_sum: tile MMAs, carried chains, warp/CTA/grid collapse,
and for N > 1 the NCCL allreduce of the per-GPU fp64 partials plus the final
rounding) over one batch of synthetic input resident in HBM.

Workloads (DESIGN.md §"Input recipe"):
  c3 (default): N = 1: n = 2^30 fp16 uniform[-1,1] (BASELINE config 3);
      N > 1: config 4, a fixed global n = 2^33 cut into N contiguous shards
      (strong scaling; --n-per-rank switches to weak scaling for tests).
  c5: 2^20 CSR segments, log-uniform lengths in [256, 65536] (config 5).

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--algo A]
                        [--workload c3|c5] [--impl ours|reference]
For N > 1 run under torchrun (one process per GPU, NCCL).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "reduction throughput Gelem/s and HBM GB/s (% of 8 TB/s roofline) at 1/2/4/8 B200"
N_C3 = 1 << 30  # BASELINE config 3: one GPU
N_C4 = 1 << 33  # BASELINE config 4: sharded over 2/4/8 GPUs (strong scaling)


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _traffic(algo: str, workload: str):
    """dram bytes per launch from the committed ncu --set full capture, if any."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(f"{workload}:{algo}")
    except Exception:
        return None


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.trace = []  # (perf_counter, sm_mhz, reason mask)
        self.window = None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = self._handle_for_cuda_device(pynvml, index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    @staticmethod
    def _handle_for_cuda_device(pynvml, index: int):
        """NVML handle of the CUDA device `index`, matched by UUID or PCI address
        (CUDA's device order need not be NVML's, e.g. without
        CUDA_DEVICE_ORDER=PCI_BUS_ID); the index only as a last resort."""
        import torch

        p = torch.cuda.get_device_properties(index)
        try:  # UUID first (survives virtualised PCI addresses), then PCI address
            return pynvml.nvmlDeviceGetHandleByUUID(f"GPU-{p.uuid}".encode())
        except Exception:
            pass
        try:
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            return pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:
            return pynvml.nvmlDeviceGetHandleByIndex(index)

    def _run(self):
        while not self._stop.is_set():
            try:
                mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.trace.append((time.perf_counter(), mhz, mask))
            except Exception:
                pass
            time.sleep(0.0002)  # ~6 ms timed regions (20 steps): sample densely

    def set_window(self, t0: float, t1: float):
        """Keep the samples taken inside the timed region [t0, t1] (wall clock);
        if the region was too short for any, the nearest sample on each side."""
        inside = [s for s in self.trace if t0 <= s[0] <= t1]
        if not inside and self.trace:
            before = [s for s in self.trace if s[0] < t0][-1:]
            after = [s for s in self.trace if s[0] > t1][:1]
            inside = before + after
        self.window = (t1 - t0) * 1e3
        self.samples = [s[1] for s in inside]
        for _, _, mask in inside:
            for bit, name in self.REASONS.items():
                if mask & bit and bit != 0x1:
                    self.reasons.add(name)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "timed_region_ms": self.window, "source": "NVML, sampled every ~0.2 ms + call time"}


def wait_for_cuda_driver(max_wait_s: float = 90.0) -> None:
    """Probe cuInit in a child process until it succeeds (bounded).  A shared
    GPU box was seen once to refuse driver initialisation for a moment right
    after another process released the GPU; a failed cuInit inside this
    process would not be retried, so it is probed outside first."""
    import subprocess

    probe = "import ctypes, sys; sys.exit(ctypes.CDLL('libcuda.so.1').cuInit(0))"
    t0 = time.time()
    while True:
        r = subprocess.run([sys.executable, "-c", probe], capture_output=True)
        if r.returncode == 0:
            return
        if time.time() - t0 > max_wait_s:
            print(f"warning: cuInit still failing (rc {r.returncode}) after {max_wait_s:.0f} s",
                  file=sys.stderr)
            return
        time.sleep(3.0)


def _cpu_count():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_oracle_leg(bits_sample, threads: int, want_sum: bool = False):
    """Time the exact oracle (as it stands) on a host sample; returns (Gelem/s,
    seconds) and, with want_sum, the oracle's ExactSum too."""
    import oracle

    t0 = time.perf_counter()
    es = oracle.exact_sum_fp16(bits_sample, threads=threads)
    dt = time.perf_counter() - t0
    if want_sum:
        return bits_sample.size / dt / 1e9, dt, es
    return bits_sample.size / dt / 1e9, dt


def c3c4_workload(world: int, n_total: int, dtype: str, weak: bool) -> str:
    """config.workload of the flat reduction lines (both arms use it): C3 at
    N = 1, C4 (sharded) at N > 1."""
    lg = n_total.bit_length() - 1
    lgs = f"2^{lg}" if n_total == 1 << lg else str(n_total)
    if world == 1:
        return f"c3: sum of n={lgs} {dtype} uniform[-1,1] on one GPU"
    return (f"c4: sharded sum, n={lgs} {dtype} uniform[-1,1] over {world} GPUs "
            f"({'weak: fixed per rank' if weak else 'strong: fixed global n'})")


def run_reference(args):
    """--impl reference: the CPU oracle on the box's host cores (tier rule: the
    reference arm is the oracle), on the same workload as our arm's line for
    this N: C3 (2^30) at N = 1, C4 (the whole 2^33 array, seed C4) at N > 1;
    every step reduces all of it.  Rank 0 only; other ranks exit without
    work."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import numpy as np

    import tcr_inputs as gen

    # generated on the host in parallel chunks (untimed)
    from concurrent.futures import ThreadPoolExecutor

    weak = args.n_per_rank is not None
    sample = (args.n_per_rank * world if weak else
              args.n_total if args.n_total is not None else (N_C3 if world == 1 else N_C4))
    seed = gen.SEED_C3 if world == 1 else gen.SEED_C4
    threads = _cpu_count()
    bits = np.empty(sample, dtype=np.uint16)
    step = 1 << 22

    def fill(lo):
        bits[lo:lo + step] = gen.generate(seed, lo, min(step, sample - lo), gen.UNIFORM_PM1)

    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(fill, range(0, sample, step)))
    for _ in range(max(args.warmup, 0)):
        cpu_oracle_leg(bits, threads)
    times = [cpu_oracle_leg(bits, threads)[1] for _ in range(args.steps)]
    tot = sum(times)
    value = sample * args.steps / tot / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Gelem/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
        "scaling": "strong" if world > 1 and not weak else "weak",
        "vs_baseline": None, "dtype": "int128", "data": "synthetic",
        "config": {"workload": c3c4_workload(world, sample, "f16", weak),
                   "sample_elems_per_step": sample, "n_total": sample},
        "cpu_baseline": {"value": value, "unit": "Gelem/s", "cores": threads, "kind": "oracle",
                         "sample": f"all {sample} elements of the workload per step, "
                                   f"exact int128 oracle, {threads} threads", **_host_info()},
        "e2e": {"value": value, "unit": "Gelem/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    del np


def _host_info():
    """CPU model and host RAM of the box (BASELINE.md §3's CPU-baseline plan)."""
    model, ram = None, None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemTotal"):
                    ram = round(int(line.split()[1]) / 2 ** 20, 1)
                    break
    except OSError:
        pass
    return {"cpu_model": model, "host_ram_gib": ram, "host_cpus": _cpu_count()}


def _exact_check(g: float, es, oracle) -> dict:
    """The timed result g against the oracle's exact sum of the same array."""
    units = es.A * es.unit / oracle.UNIT  # sum |x| in units of 2^-24
    return {"gpu_f32": g, "exact_f64": es.f64(),
            "err_units_2^-24_sum_abs": (float(oracle.error_units(g, es) / units) if units else 0.0),
            "within_2^-20_sum_abs": bool(oracle.within_tolerance(g, es)),
            "bitwise_equal_rne_exact": g == es.f32()}


def cpu_legs_single(args, x, n, out32, dev, gen, np, torch):
    """N = 1: the oracle (as it stands) on the host cores over the workload's
    own elements -- all threads, repeated until ~cpu_seconds; one thread on a
    2^26 prefix; the D2H time of the sample reported separately -- and the
    timed result checked against the exact sum of the same array."""
    import oracle

    sample = min(n, 1 << 30)
    t0 = time.perf_counter()
    if x.element_size() == 2 and args.dtype == "f16":
        bits = x[:sample].view(torch.int16).cpu().numpy().view(np.uint16)
    else:  # bf16 / fp8 runs: time the binary16 oracle on the c3 stream of the same length
        bits = gen.generate_tensor(gen.SEED_C3, 0, sample, gen.UNIFORM_PM1,
                                   device=dev).view(torch.int16).cpu().numpy().view(np.uint16)
    d2h_ms = (time.perf_counter() - t0) * 1e3
    threads = _cpu_count()
    done, spent, passes, es = 0, 0.0, 0, None
    while spent < args.cpu_seconds or passes == 0:
        _, dt, es = cpu_oracle_leg(bits, threads, want_sum=True)
        done += bits.size
        spent += dt
        passes += 1
    one = bits[:min(bits.size, 1 << 26)]
    done1, spent1, passes1 = 0, 0.0, 0
    while spent1 < args.cpu_seconds / 4 or passes1 == 0:
        _, dt = cpu_oracle_leg(one, 1)
        done1 += one.size
        spent1 += dt
        passes1 += 1
    cpu = {"value": done / spent / 1e9, "unit": "Gelem/s", "cores": threads, "kind": "oracle",
           "sample": f"{passes} passes over the first {sample} elements of the workload "
                     f"({'all' if sample == n else 'part'} of it), exact int128 oracle, "
                     f"{threads} threads, {spent:.1f} s",
           "one_thread": {"value": done1 / spent1 / 1e9, "unit": "Gelem/s", "cores": 1,
                          "sample": f"{passes1} passes over the first {one.size} elements, "
                                    f"{spent1:.1f} s"},
           "d2h_ms": d2h_ms, "d2h_bytes": int(bits.nbytes),
           "d2h_note": "copy of the oracle's sample from HBM to pageable host memory, "
                       "not included in value",
           **_host_info()}
    check = None
    if out32 is None:  # c5: the segment outputs are checked by the tests, not here
        pass
    elif args.dtype == "f16" and sample == n:
        check = _exact_check(float(out32.item()), es, oracle)
    elif args.dtype != "f16":  # the dtype's own exact oracle over the timed array
        raw = x.view(torch.uint8).cpu().numpy()
        if args.dtype == "bf16":
            esd = oracle.ExactSum(0, 0, unit_exp=-133)
            b16 = raw.view(np.uint16)
            for lo in range(0, b16.size, 1 << 26):
                esd = esd + oracle.exact_sum_bf16(b16[lo:lo + (1 << 26)])
        else:
            esd = oracle.exact_sum_fp8(raw, oracle.FP8_E4M3 if args.dtype == "e4m3"
                                       else oracle.FP8_E5M2)
        check = _exact_check(float(out32.item()), esd, oracle)
        del raw
    del bits
    return cpu, check


def _limbs(v: int) -> list:
    """A (possibly negative) Python int as three int64 limbs, base 2^40 (the
    top limb signed), so that limb-wise integer sums across ranks are exact."""
    m = (1 << 40) - 1
    return [v & m, (v >> 40) & m, v >> 80]


def cpu_legs_sharded(args, x, n, n_total, out32, dev, world, np, torch, dist):
    """N > 1: every rank copies its shard back and runs the exact oracle on
    it (the ranks share the host's cores, threads split evenly); the exact
    shard sums add exactly (homomorphism) through an int64
    limb allreduce; the timed result is checked against the exact total.
    cpu_baseline = the whole C4 array reduced by the oracle on the host
    (all ranks concurrently, time = max over ranks)."""
    import oracle

    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    threads = max(1, _cpu_count() // max(1, local_world))
    t0 = time.perf_counter()
    if args.dtype == "f16":
        bits = x.view(torch.int16).cpu().numpy().view(np.uint16)
    else:  # time the binary16 oracle on the c4 stream of the same shard
        bits = None
    d2h_ms = (time.perf_counter() - t0) * 1e3
    if bits is None:
        return None, None
    t0 = time.perf_counter()
    es = oracle.exact_sum_fp16(bits, threads=threads)
    dt = time.perf_counter() - t0
    del bits
    v = torch.tensor(_limbs(es.T) + _limbs(es.A) + [es.n_nan, es.n_pinf, es.n_ninf],
                     dtype=torch.int64, device=dev)
    dist.all_reduce(v)
    tm = torch.tensor([dt, d2h_ms], dtype=torch.float64, device=dev)
    dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    a = [int(t) for t in v.tolist()]
    total = oracle.ExactSum(a[0] + (a[1] << 40) + (a[2] << 80), a[3] + (a[4] << 40) + (a[5] << 80),
                            a[6], a[7], a[8])
    dt_max, d2h_max = tm.tolist()
    cpu = {"value": n_total / dt_max / 1e9, "unit": "Gelem/s", "cores": threads * world,
           "kind": "oracle",
           "sample": f"the whole {n_total}-element C4 array, each of {world} ranks reducing its "
                     f"own shard on {threads} host threads concurrently (max over ranks "
                     f"{dt_max:.2f} s), exact int128 oracle",
           "d2h_ms": d2h_max, "d2h_bytes": 2 * n_total,
           "d2h_note": "max over ranks of the shard copy to pageable host memory, not in value",
           **_host_info()}
    return cpu, _exact_check(float(out32.item()), total, oracle)


def one_gpu_c4_time(args, rank, n_total, algo, dev, gen, torch, tcr):
    """T_1 for strong scaling: rank 0 alone reduces the WHOLE C4 array on its
    GPU with the same kernel (same warm-up / step counts, back-to-back
    launches between CUDA events).  Other ranks return None."""
    if rank != 0:
        return None
    if args.dtype != "f16":
        return {"skipped": "binary16 (C4) only"}
    free, _ = torch.cuda.mem_get_info(dev)
    if 2 * n_total > free * 0.9:
        return {"skipped": f"needs {2 * n_total} B, {free} B free"}
    xa = gen.generate_tensor(gen.SEED_C4, 0, n_total, gen.UNIFORM_PM1, device=dev)
    o = torch.empty(1, dtype=torch.float32, device=dev)
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        for _ in range(args.warmup):
            tcr.tcr_reduce_sum_ex(xa, out_f32=o, algo=algo, stream=s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(args.steps):
            tcr.tcr_reduce_sum_ex(xa, out_f32=o, algo=algo, stream=s)
        e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    del xa
    return {"n": n_total, "ms_per_step": ms, "value": n_total / (ms * 1e-3) / 1e9,
            "unit": "Gelem/s", "what": "one GPU (rank 0) reducing the whole C4 array, same kernel"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--algo", default="default",
                    choices=["default", "mma_sync", "tcgen05", "shuffle", "bulk", "exact"])
    ap.add_argument("--workload", default="c3", choices=["c3", "c5"])
    ap.add_argument("--dtype", default="f16", choices=["f16", "bf16", "e4m3", "e5m2"],
                    help="input element type (bf16 / fp8 = NEXT-4; c3 workload, non-exact algos)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--combine", default="auto", choices=["auto", "nccl", "peer"],
                    help="c3/c4 cross-GPU combine: one NCCL allreduce of the fp64 partials, "
                         "or the fused in-kernel NVLink mailbox combine (NEXT-2, peer.py); "
                         "auto = peer for N > 1 when its setup and a check against the NCCL "
                         "combine pass on every rank, else nccl")
    ap.add_argument("--n-total", type=int, default=None,
                    help="global element count (default: 2^30 = C3 at N=1, 2^33 = C4 at N>1)")
    ap.add_argument("--n-per-rank", type=int, default=None,
                    help="weak-scaling override: this many elements per rank (tests)")
    ap.add_argument("--no-t1", action="store_true",
                    help="N>1: skip rank 0's one-GPU timing of the whole C4 array")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="CPU-oracle baseline: repeat passes until this much CPU time")
    ap.add_argument("--unroll", type=int, help="TCR_CFG_UNROLL (mma_sync/shuffle)")
    ap.add_argument("--bps", type=int, help="TCR_CFG_BLOCKS_PER_SM")
    ap.add_argument("--chain", type=int, help="TCR_CFG_CHAIN (carried chain K, tiles)")
    ap.add_argument("--stages", type=int, help="TCR_CFG_TC05_STAGES")
    ap.add_argument("--stage-kb", type=int, help="TCR_CFG_TC05_STAGE_KB")
    ap.add_argument("--slots", type=int, help="TCR_CFG_TC05_SLOTS")
    ap.add_argument("--tc-chain", type=int, help="TCR_CFG_TC05_CHAIN")
    ap.add_argument("--ctas", type=int, help="TCR_CFG_TC05_CTAS_PER_SM")
    ap.add_argument("--prefetch", type=int, help="TCR_CFG_TC05_PREFETCH")
    ap.add_argument("--split", type=int, help="TCR_CFG_TC05_SPLIT")
    ap.add_argument("--interleave", type=int, help="TCR_CFG_TC05_INTERLEAVE")
    ap.add_argument("--bulk-stages", type=int, help="TCR_CFG_BULK_STAGES")
    ap.add_argument("--bulk-kb", type=int, help="TCR_CFG_BULK_STAGE_KB")
    ap.add_argument("--bulk-ctas", type=int, help="TCR_CFG_BULK_CTAS_PER_SM")
    ap.add_argument("--exact-unroll", type=int, help="TCR_CFG_EXACT_UNROLL")
    ap.add_argument("--exact-bps", type=int, help="TCR_CFG_EXACT_BLOCKS_PER_SM")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1903_03640_b200 as tcr
    import tcr_inputs as gen

    for key, val in ((tcr.TCR_CFG_UNROLL, args.unroll), (tcr.TCR_CFG_BLOCKS_PER_SM, args.bps),
                     (tcr.TCR_CFG_CHAIN, args.chain), (tcr.TCR_CFG_TC05_STAGES, args.stages),
                     (tcr.TCR_CFG_TC05_STAGE_KB, args.stage_kb), (tcr.TCR_CFG_TC05_SLOTS, args.slots),
                     (tcr.TCR_CFG_TC05_CHAIN, args.tc_chain), (tcr.TCR_CFG_TC05_CTAS_PER_SM, args.ctas),
                     (tcr.TCR_CFG_TC05_PREFETCH, args.prefetch), (tcr.TCR_CFG_TC05_SPLIT, args.split),
                     (tcr.TCR_CFG_TC05_INTERLEAVE, args.interleave),
                     (tcr.TCR_CFG_BULK_STAGES, args.bulk_stages),
                     (tcr.TCR_CFG_BULK_STAGE_KB, args.bulk_kb),
                     (tcr.TCR_CFG_BULK_CTAS_PER_SM, args.bulk_ctas),
                     (tcr.TCR_CFG_EXACT_UNROLL, args.exact_unroll),
                     (tcr.TCR_CFG_EXACT_BLOCKS_PER_SM, args.exact_bps)):
        if val is not None:
            tcr.tcr_set_config(key, val)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # Test hook (never used for a reported number): TCR_BENCH_SHARED_GPU=1 maps
    # every rank to cuda:0 and uses gloo, to exercise the N > 1 code path on a
    # one-GPU box.  The ranks' kernels are independent (nothing on the device
    # waits for a peer); the allreduce runs on the host.
    shared_gpu = os.environ.get("TCR_BENCH_SHARED_GPU") == "1"
    if shared_gpu:
        local = 0
    wait_for_cuda_driver()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.Stream(dev)
    exact = args.algo == "exact"
    if args.dtype != "f16" and args.workload != "c3":
        raise SystemExit("--dtype bf16/e4m3/e5m2 supports the c3 workload")
    algo = tcr.ALGOS["default" if exact else args.algo]
    peak, peak_src = _peaks()
    peer, combine_note = None, None
    peer_cfg = (args.workload == "c3" and args.dtype == "f16"
                and args.algo in ("default", "mma_sync", "tcgen05", "shuffle", "exact"))
    if args.combine == "peer":
        if not peer_cfg:
            raise SystemExit("--combine peer supports the f16 c3/c4 workload with mma_sync / "
                             "shuffle / exact")
        if shared_gpu and world > 1:
            raise SystemExit("--combine peer makes the ranks' kernels wait on one another: "
                             "never on one shared GPU")
    if args.combine == "peer" or (args.combine == "auto" and world > 1 and not shared_gpu
                                  and peer_cfg):
        from paper_1903_03640_b200.peer import PeerGroup

        try:
            peer = PeerGroup()
        except Exception as e:  # e.g. no CUDA IPC between these devices
            if args.combine == "peer":
                raise
            peer, combine_note = None, f"peer setup failed ({e}); NCCL combine used"
        if world > 1:  # every rank must take the same combine
            ok = torch.tensor([1 if peer is not None else 0], dtype=torch.int32, device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if ok.item() == 0 and peer is not None:
                peer, combine_note = None, "peer setup failed on another rank; NCCL combine used"
        if peer is not None and not exact:
            algo = tcr.ALGOS[args.algo]  # "default": by shard size inside the library

    # ---------------- inputs (untimed), resident in HBM ----------------
    if args.workload == "c3":
        from paper_1903_03640_b200.sharded import shard_range

        # N = 1: C3 (2^30 on one GPU).  N > 1: C4, a FIXED global n = 2^33
        # cut into contiguous shards (strong scaling); --n-per-rank
        # (tests) switches to weak scaling with that many elements per rank.
        weak = args.n_per_rank is not None
        n_total = (args.n_per_rank * world if weak else
                   args.n_total if args.n_total is not None else (N_C3 if world == 1 else N_C4))
        lo, hi = shard_range(n_total, world, rank)
        n = hi - lo
        seed = gen.SEED_C3 if world == 1 else gen.SEED_C4
        if args.dtype in ("e4m3", "e5m2"):
            fmt8 = gen.FP8_E4M3 if args.dtype == "e4m3" else gen.FP8_E5M2
            x = gen.generate_tensor_fp8(seed, lo, n, gen.UNIFORM_PM1, fmt8, device=dev)
        else:
            x = gen.generate_tensor(seed, lo, n, gen.UNIFORM_PM1, device=dev,
                                    bf16=args.dtype == "bf16")
        bytes_per_step = x.element_size() * n
        elems_per_step = n
        job_elems_per_step = n_total
        job_bytes_per_step = x.element_size() * n_total
        workload = c3c4_workload(world, n_total, args.dtype, weak)
    else:
        from paper_1903_03640_b200.sharded import segment_shard

        S_all = 1 << 20
        lens = gen.loguniform_lengths(gen.SEED_C5, S_all)
        off_all = gen.offsets_from_lengths(lens)
        # N > 1: whole segments sharded by element count (no collective; strong scaling)
        j0, j1 = segment_shard(off_all, world, rank)
        S = j1 - j0
        off = off_all[j0:j1 + 1] - off_all[j0]
        n = int(off[-1])
        x = gen.generate_tensor(gen.SEED_C5, int(off_all[j0]), n, gen.UNIFORM_PM1, device=dev)
        toff = torch.from_numpy(off).to(dev)
        seg_out = torch.empty(max(S, 1), dtype=torch.float32, device=dev)
        bytes_per_step = 2 * n + 8 * (S + 1) + 4 * S
        elems_per_step = n
        job_elems_per_step = int(off_all[-1])
        job_bytes_per_step = 2 * job_elems_per_step + 8 * (S_all + world) + 4 * S_all
        workload = "c5: 2^20 segments, log-uniform lengths in [256, 65536], fp16 uniform[-1,1]" + (
            f", segments sharded over {world} GPUs" if world > 1 else "")
    out32 = torch.empty(1, dtype=torch.float32, device=dev)
    out64 = torch.empty(1, dtype=torch.float64, device=dev)
    dtype_code = {"f16": tcr.TCR_DTYPE_F16, "bf16": tcr.TCR_DTYPE_BF16,
                  "e4m3": tcr.TCR_DTYPE_E4M3, "e5m2": tcr.TCR_DTYPE_E5M2}[args.dtype]
    # exact state: 6 int64 limbs (binary16 / fp8) or 27 (bfloat16), integer-summable
    exact_state = torch.empty(tcr.TCR_EXACT_BF16_ACC_WORDS if args.dtype == "bf16"
                       else tcr.TCR_EXACT_ACC_WORDS, dtype=torch.int64, device=dev)
    torch.cuda.synchronize()

    if peer is not None and world > 1:
        # check the fused combine against the NCCL combine once, on every rank
        ref64 = torch.empty(1, dtype=torch.float64, device=dev)
        p64 = torch.empty(1, dtype=torch.float64, device=dev)
        with torch.cuda.stream(stream):
            if exact:  # exact: the fused limb combine must equal the NCCL limb allreduce bitwise
                tcr.tcr_reduce_sum_exact(x, acc=exact_state, stream=stream)
                dist.all_reduce(exact_state)
                tcr.tcr_exact_finalize(exact_state, out_f64=ref64, stream=stream)
                peer.reduce_sum_exact(x, out_f64=p64, stream=stream)
            else:
                tcr.tcr_reduce_sum_ex(x, out_f64=ref64, algo=algo, stream=stream)
                dist.all_reduce(ref64)
                peer.reduce_sum(x, out_f64=p64, algo=algo, stream=stream)
        torch.cuda.synchronize()
        r, g = ref64.item(), p64.item()
        tol = 0.0 if exact else 1e-9 * max(1.0, abs(r))
        good = math.isfinite(g) and abs(g - r) <= tol and not peer.timed_out()
        ok = torch.tensor([1 if good else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if ok.item() == 0:
            if args.combine == "peer":
                raise SystemExit(f"fused peer combine disagrees with NCCL: {g!r} vs {r!r}")
            peer.close()
            peer, combine_note = None, "peer combine check failed; NCCL combine used"
            algo = tcr.ALGOS["default" if exact else args.algo]

    def step(ev_k0=None, ev_k1=None):
        with torch.cuda.stream(stream):
            if ev_k0 is not None:
                ev_k0.record(stream)
            if args.workload == "c5":
                tcr.tcr_reduce_sum_segmented(x, toff, seg_out, num_segments=S, stream=stream)
            elif peer is not None and exact:  # exact sum + limb combine in ONE launch
                peer.reduce_sum_exact(x, out_f32=out32, stream=stream)
            elif peer is not None:  # reduction + cross-GPU combine in ONE launch
                peer.reduce_sum(x, out_f32=out32, algo=algo, stream=stream)
            elif exact:  # N = 1: the rounded result only (one kernel); N > 1: the mergeable state
                tcr.tcr_reduce_sum_exact_ex(x, acc=exact_state if world > 1 else None,
                                            out_f32=out32 if world == 1 else None, stream=stream)
            elif world == 1:
                tcr.tcr_reduce_sum_ex(x, out_f32=out32, algo=algo, stream=stream)
            else:
                tcr.tcr_reduce_sum_ex(x, out_f64=out64, algo=algo, stream=stream)
            if ev_k1 is not None:
                ev_k1.record(stream)
            if args.workload == "c3" and world > 1 and peer is None:
                if exact:  # integer limbs: the allreduce is exact, result independent of N
                    dist.all_reduce(exact_state)
                    tcr.tcr_exact_finalize_ex(exact_state, dtype_code, out_f32=out32, stream=stream)
                else:
                    dist.all_reduce(out64)  # the paper's distributed merge, over NVLink
                    tcr.tcr_round_f64_to_f32(out64, out32, stream=stream)

    # ---------------- end to end through the public API with host buffers ----------------
    # Runs BEFORE the device-resident timed region: a fresh process's first
    # ~25 launches run 2-10 % slower while the GPU settles (profiles/r02/
    # warm_fresh.txt), so the e2e leg also serves as the settling phase.
    e2e = None
    if args.workload == "c3" and args.e2e_steps > 0:
        # the step's input bits in pinned host memory (any element type)
        esz = x.element_size()
        host = torch.empty(n * esz, dtype=torch.uint8, pin_memory=True)
        host.copy_(x.view(torch.uint8).reshape(-1))
        res_t = torch.empty(1, dtype=torch.float32, device=dev)
        hs = torch.cuda.Stream(dev)
        for _ in range(3):  # warm-up (a fresh box's first call ran at 85 % of the PCIe rate)
            tcr.tcr_reduce_sum_host_ex(host, dtype_code, n=n, stream=hs.cuda_stream)
        if world > 1:
            dist.barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(hs)
        for _ in range(args.e2e_steps):
            # H2D + reduce + D2H through the public host entry point
            g = tcr.tcr_reduce_sum_host_ex(host, dtype_code, n=n, stream=hs.cuda_stream)
            if world > 1:
                res_t.fill_(g)
                dist.all_reduce(res_t)
        ev1.record(hs)
        torch.cuda.synchronize()
        e_ms = ev0.elapsed_time(ev1)
        if world > 1:
            t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = t.item()
        e2e = {"value": world * n * args.e2e_steps / (e_ms * 1e-3) / 1e9, "unit": "Gelem/s",
               "h2d_bytes_per_step": esz * n, "d2h_bytes_per_step": 4, "steps": args.e2e_steps,
               "api": "tcr_reduce_sum_host_ex (pinned host input, chunked H2D inside the call)"}
        del host

    clk = ClockSampler(torch.cuda.current_device()).__enter__()
    nvtx = torch.cuda.nvtx  # ranges for profiler filtering (ncu --nvtx); host-side only
    nvtx.range_push("tcr.warmup")
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    nvtx.range_pop()

    K = args.steps
    # A step that is ONE launch of the dominant kernel (N = 1, or the fused
    # peer combine) runs back to back with no events inside the timed region:
    # the kernel's average launch duration is then the region / K (launch
    # gaps included -- a per-step event pair would add its own gap, ~3 %).
    # A step with an NCCL call keeps one event pair around the kernel.
    single_launch_step = world == 1 or peer is not None
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(0 if single_launch_step else K)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = tcr.tcr_launch_count()
    w0 = time.perf_counter()
    nvtx.range_push("tcr.timed")
    t_start.record(stream)
    for i in range(K):
        step(*kev[i]) if kev else step()
    t_end.record(stream)
    torch.cuda.synchronize()
    w1 = time.perf_counter()
    nvtx.range_pop()
    time.sleep(0.01)
    clk.__exit__(None, None, None)
    clk.set_window(w0, w1)
    launches = tcr.tcr_launch_count() - launches0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    total_ms = t_start.elapsed_time(t_end)
    if single_launch_step:
        if launches != K:
            raise SystemExit(f"expected one launch per step, counted {launches} for {K} steps")
        kern_ms = total_ms / K
    else:
        kern_ms = statistics.mean(a.elapsed_time(b) for a, b in kev)
    if world > 1:
        t = torch.tensor([total_ms, kern_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, kern_ms = t.tolist()

    # correctness spot-check of the last step's result is done by the tests;
    # here only record the value for the log
    result = float(out32.item()) if args.workload == "c3" else float(seg_out[0].item())

    value = job_elems_per_step * K / (total_ms * 1e-3) / 1e9  # Gelem/s, whole job
    achieved = bytes_per_step / (kern_ms * 1e-3) / 1e9              # GB/s of the dominant kernel
    if args.algo != "default":
        algo_name = args.algo
    elif args.workload == "c5":
        algo_name = "mma_sync"  # the segmented MMA kernels
    else:  # what TCR_ALGO_DEFAULT resolved to for this rank's input size
        algo_name = {1: "mma_sync", 2: "tcgen05", 3: "shuffle", 4: "bulk"}[
            tcr.tcr_default_algo(n, dtype_code)]

    cpu, check, t1 = None, None, None
    if not args.no_cpu_baseline:
        if world == 1:
            cpu, check = cpu_legs_single(args, x, n, out32 if args.workload == "c3" else None,
                                         dev, gen, np, torch)
        elif args.workload == "c3":
            cpu, check = cpu_legs_sharded(args, x, n, n_total, out32, dev, world, np, torch, dist)
    if args.workload == "c3" and world > 1 and not args.no_t1:
        t1 = one_gpu_c4_time(args, rank, n_total, algo, dev, gen, torch, tcr)
        dist.barrier()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Gelem/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": total_ms / K, "higher_is_better": True,
            "scaling": ("strong" if world > 1 and not (args.workload == "c3" and weak)
                        else "weak"),
            "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic (splitmix64-seeded, generated on the device)",
            "config": {"workload": workload, "algo": algo_name, "n_per_rank": n,
                       "knobs": {k: tcr.tcr_get_config(v) for k, v in (
                           ("unroll", tcr.TCR_CFG_UNROLL), ("blocks_per_sm", tcr.TCR_CFG_BLOCKS_PER_SM),
                           ("chain", tcr.TCR_CFG_CHAIN), ("tc05_stages", tcr.TCR_CFG_TC05_STAGES),
                           ("tc05_stage_kb", tcr.TCR_CFG_TC05_STAGE_KB), ("tc05_slots", tcr.TCR_CFG_TC05_SLOTS),
                           ("tc05_chain", tcr.TCR_CFG_TC05_CHAIN), ("tc05_ctas", tcr.TCR_CFG_TC05_CTAS_PER_SM),
                           ("tc05_prefetch", tcr.TCR_CFG_TC05_PREFETCH), ("tc05_split", tcr.TCR_CFG_TC05_SPLIT),
                           ("tc05_interleave", tcr.TCR_CFG_TC05_INTERLEAVE),
                           ("tc05_dynamic", tcr.TCR_CFG_TC05_DYNAMIC),
                           ("tc05_dyn_min_run", tcr.TCR_CFG_TC05_DYN_MIN_RUN),
                           ("default_algo", tcr.TCR_CFG_DEFAULT_ALGO))},
                       "n_total": job_elems_per_step, "l2": "inputs larger than L2 (no flush needed)",
                       "combine": ("fused in-kernel NVLink mailbox combine (peer.py)" if peer
                                   else "NCCL allreduce of fp64 partials") if world > 1 or peer
                                  else "none (single GPU)",
                       "combine_note": combine_note,
                       "parallelism": f"dp{world}" if world > 1 else "single"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": _traffic(
                             algo_name,
                             args.workload if args.dtype == "f16" else f"{args.workload}-{args.dtype}"),
                         "peak_source": peak_src, "kernel_ms": kern_ms,
                         "kernel_ms_method": ("timed region / K (one launch per step, back to back)"
                                              if single_launch_step else
                                              "mean of per-step CUDA event pairs around the kernel"),
                         "algorithmic_bytes_per_launch": bytes_per_step},
            "hbm_gbs": job_bytes_per_step * K / (total_ms * 1e-3) / 1e9,
            "frac_of_8tbs": job_bytes_per_step * K / (total_ms * 1e-3) / (world * 8e12),
            "cpu_baseline": cpu,
            "check": check,
            "t1": t1,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "result": result,
        }
        if shared_gpu:
            line["test_mode"] = "shared-gpu gloo (not a measurement)"
        print(json.dumps(line), flush=True)
    if peer is not None:
        if peer.timed_out():
            print(f"warning: rank {rank}: a fused combine timed out", file=sys.stderr, flush=True)
        peer.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
