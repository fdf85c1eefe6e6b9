"""Exact kernel vs tcgen05 default: per-launch time and SM clock (NVML)
during sustained blocks of launches at 2^30 and 2^32 -- is the exact kernel's
per-element slowdown at 2^32 a power / clock effect?"""
import statistics
import sys
import threading
import time

import pynvml
import torch

sys.path.insert(0, ".")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
out = torch.empty(1, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()


def run(f, k):
    clocks, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            clocks.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            pw = pynvml.nvmlDeviceGetPowerUsage(h)
            clocks.append(-pw // 1000)
            time.sleep(0.002)

    th = threading.Thread(target=sample)
    with torch.cuda.stream(s):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        th.start()
        a.record(s)
        for _ in range(k):
            f()
        b.record(s)
    torch.cuda.synchronize()
    stop.set()
    th.join()
    mhz = [c for c in clocks if c > 0]
    w = [-c for c in clocks if c <= 0]
    return a.elapsed_time(b) * 1e3 / k, statistics.median(mhz) if mhz else 0, max(w) if w else 0


for lg, k in ((30, 200), (32, 50)):
    n = 1 << lg
    x = gen.generate_tensor(gen.SEED_C3, 0, n, gen.UNIFORM_PM1)
    fe = lambda: tcr.tcr_reduce_sum_exact(x, out_f32=out, stream=s)  # noqa: E731
    ft = lambda: tcr.tcr_reduce_sum_algo(x, out_f32=out, algo="tcgen05", stream=s)  # noqa: E731
    fm = lambda: tcr.tcr_reduce_sum_algo(x, out_f32=out, algo="mma_sync", stream=s)  # noqa: E731
    for name, f in (("exact", fe), ("tcgen05", ft), ("mma_sync", fm), ("exact", fe)):
        run(f, 5)
        t, mhz, w = run(f, k)
        print(f"2^{lg} {name:9s} {t:9.2f} us/launch {2 * n / t / 1e3:6.0f} GB/s  SM {mhz:.0f} MHz  max {w:.0f} W",
              flush=True)
    del x
    torch.cuda.empty_cache()
