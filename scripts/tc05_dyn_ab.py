"""r02 §16: the tcgen05 dynamic tail (TCR_CFG_TC05_DYNAMIC) against mma.sync
and the static tcgen05 partition, interleaved on one box.
  back to back: rounds of 20 launches between two events (the driver's bench
                shape), median of 8 interleaved rounds;
  isolated:     each launch queued behind a 40 us spin kernel, one event pair
                around the launch alone (device time, host launch cost
                outside), median of 30;
  warm graph:   CUDA graph of 100 launches (small n).
Usage: DYNS="0 10 25" python scripts/tc05_dyn_ab.py [log2 sizes, default 26 27 28 30 32 33]"""
import statistics
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402
from c2_compare_lib import graph_time  # noqa: E402

sizes = [int(a) for a in sys.argv[1:]] or [26, 27, 28, 30, 32, 33]
import os  # noqa: E402

dyns = [int(v) for v in os.environ.get("DYNS", "0 10 25 50").split()]
arms = [("mma_sync", "mma_sync", None)] + [(f"tc05 dyn{d}", "tcgen05", d) for d in dyns]
out = torch.empty(1, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()


def setup(dyn):
    if dyn is not None:
        tcr.tcr_set_config(tcr.TCR_CFG_TC05_DYNAMIC, dyn)


def b2b(x, algo, k=20):
    with torch.cuda.stream(s):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(k):
            tcr.tcr_reduce_sum_ex(x, out_f32=out, algo=algo, stream=s)
        b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / k


def isolated(x, algo):
    with torch.cuda.stream(s):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(int(40e-6 * 1.9e9))
        a.record(s)
        tcr.tcr_reduce_sum_ex(x, out_f32=out, algo=algo, stream=s)
        b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3


dtype = os.environ.get("DTYPE", "f16")
es = 1 if dtype in ("e4m3", "e5m2") else 2
for lg in sizes:
    n = 1 << lg
    if es == 1:
        x = gen.generate_tensor_fp8(gen.SEED_C3, 0, n, gen.UNIFORM_PM1,
                                    gen.FP8_E4M3 if dtype == "e4m3" else gen.FP8_E5M2)
    else:
        x = gen.generate_tensor(gen.SEED_C3, 0, n, gen.UNIFORM_PM1, bf16=(dtype == "bf16"))
    for name, algo, dyn in arms:  # warm every path over this buffer
        setup(dyn)
        b2b(x, algo, 30)
    res = {name: [] for name, _, _ in arms}
    iso = {name: [] for name, _, _ in arms}
    for r in range(8):
        for name, algo, dyn in arms:
            setup(dyn)
            res[name].append(b2b(x, algo))
    for r in range(30):
        for name, algo, dyn in arms:
            setup(dyn)
            iso[name].append(isolated(x, algo))
    base = statistics.median(res["mma_sync"])
    ibase = statistics.median(iso["mma_sync"])
    print(f"{dtype} 2^{lg}: back to back (20 launches, median of 8) | isolated (behind a spin, median of 30)")
    for name, _, _ in arms:
        m, mi = statistics.median(res[name]), statistics.median(iso[name])
        print(f"  {name:12s} {m:9.2f} us {es * n / m / 1e3:6.0f} GB/s {m / base:.3f}x mma | "
              f"{mi:9.2f} us {es * n / mi / 1e3:6.0f} GB/s {mi / ibase:.3f}x mma", flush=True)
    if os.environ.get("SUSTAIN"):  # blocks of 200 launches (~60 ms at 2^30), 4 interleaved rounds
        import pynvml  # noqa: E402

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        sus = {name: [] for name, _, _ in arms}
        for r in range(4):
            for name, algo, dyn in arms:
                setup(dyn)
                t = b2b(x, algo, 200)
                sus[name].append((t, pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
        print("  sustained (blocks of 200, us per launch @ SM MHz after the block):")
        for name, _, _ in arms:
            print(f"    {name:12s} " + "  ".join(f"{t:8.2f}@{c}" for t, c in sus[name]) +
                  f"   median {statistics.median(t for t, _ in sus[name]):.2f}", flush=True)
    if lg <= 26:
        g = {}
        for name, algo, dyn in arms:
            setup(dyn)
            g[name] = statistics.median(
                graph_time(lambda: tcr.tcr_reduce_sum_ex(x, out_f32=out, algo=algo)) for _ in range(3))
        print("  warm graph: " + "  ".join(f"{k} {v:.2f} us" for k, v in g.items()), flush=True)
    del x
    torch.cuda.empty_cache()
tcr.tcr_set_config(tcr.TCR_CFG_TC05_DYNAMIC, 8)
