"""Default-path decision (r02, verdict next #5): mma.sync vs the tcgen05
kernel with the tight issue loop, interleaved on one box.
  2^30, rounds of 20 back-to-back launches (the driver's bench shape), and
  a sustained phase (blocks of 200 launches, ~0.7 s of load, alternating)
  where sw_power_cap brings the SM clock down; NVML SM clock per block.
  2^24 warm: CUDA graph of 100 launches.
tcgen05 configs: (stages, KiB, slots, chain, CTAs/SM)."""
import statistics
import sys

import pynvml
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402
from c2_compare_lib import graph_time  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
keys = (tcr.TCR_CFG_TC05_STAGES, tcr.TCR_CFG_TC05_STAGE_KB, tcr.TCR_CFG_TC05_SLOTS,
        tcr.TCR_CFG_TC05_CHAIN, tcr.TCR_CFG_TC05_CTAS_PER_SM)
arms = [("mma_sync", None), ("tcgen05 default (auto)", (4, 32, 4, 2, 0)),
        ("tcgen05 4x32 K2 1cta", (4, 32, 4, 2, 1)), ("tcgen05 2x32 K2 3cta", (2, 32, 4, 2, 3)),
        ("tcgen05 r01 4x16 3cta", (4, 16, 4, 4, 3))]
x30 = gen.generate_tensor(gen.SEED_C3, 0, 1 << 30, gen.UNIFORM_PM1)
x24 = gen.generate_tensor(gen.SEED_C2, 0, 1 << 24, gen.UNIFORM_PM1)
out = torch.empty(1, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()


def setup(cfg):
    if cfg is not None:
        for k, v in zip(keys, cfg):
            tcr.tcr_set_config(k, v)
    return "mma_sync" if cfg is None else "tcgen05"


def block(x, algo, k):
    with torch.cuda.stream(s):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(k):
            tcr.tcr_reduce_sum_algo(x, out_f32=out, algo=algo, stream=s)
        b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / k


res20 = {n: [] for n, _ in arms}
for r in range(8):
    for name, cfg in arms:
        algo = setup(cfg)
        block(x30, algo, 3)
        res20[name].append(block(x30, algo, 20))
print("2^30, 20 back-to-back launches, median of 8 interleaved rounds:")
base = statistics.median(res20["mma_sync"])
for name, _ in arms:
    m = statistics.median(res20[name])
    print(f"  {name:24s} {m:7.1f} us  {2 ** 31 / m / 1e3:6.0f} GB/s  {m / base:.3f}x mma", flush=True)

sus = {n: [] for n, _ in arms}
for r in range(4):
    for name, cfg in arms:
        algo = setup(cfg)
        t = block(x30, algo, 200)
        sus[name].append((t, pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
print("2^30 sustained (blocks of 200 launches, 4 interleaved rounds): us per launch @ SM MHz after the block")
for name, _ in arms:
    print(f"  {name:24s} " + "  ".join(f"{t:6.1f}@{c}" for t, c in sus[name]) +
          f"   median {statistics.median(t for t, _ in sus[name]):.1f}", flush=True)

print("2^24 warm (CUDA graph of 100 launches, median of 3):")
g24 = {}
for name, cfg in arms:
    algo = setup(cfg)
    g24[name] = statistics.median(graph_time(lambda: tcr.tcr_reduce_sum_algo(x24, out_f32=out, algo=algo))
                                  for _ in range(3))
for name, _ in arms:
    print(f"  {name:24s} {g24[name]:6.2f} us  {g24[name] / g24['mma_sync']:.2f}x mma", flush=True)
