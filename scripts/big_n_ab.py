"""Large-n default decision (r02): the LDG-fed mma.sync kernel vs the
TMA-fed ones (bulk: cp.async.bulk -> SMEM -> ld.shared -> mma.sync, one CTA
per SM; tcgen05 r02 default), interleaved on one box: 2^30 in rounds of 20
back-to-back launches (the driver's bench shape, 10 rounds) and a sustained
phase (blocks of 200); 2^24 / 2^26 / 2^28 warm graphs for the size rule."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402
from c2_compare_lib import graph_time  # noqa: E402

bk = (tcr.TCR_CFG_BULK_STAGES, tcr.TCR_CFG_BULK_STAGE_KB, tcr.TCR_CFG_BULK_CTAS_PER_SM)
saved = [tcr.tcr_get_config(k) for k in bk]
arms = [("mma_sync", "mma_sync", None), ("bulk 2x64 c1", "bulk", (2, 64, 1)),
        ("bulk 4x32 c1", "bulk", (4, 32, 1)), ("tcgen05", "tcgen05", None)]
out = torch.empty(1, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()


def setup(cfg):
    if cfg:
        for k, v in zip(bk, cfg):
            tcr.tcr_set_config(k, v)


def block(x, algo, k):
    with torch.cuda.stream(s):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(k):
            tcr.tcr_reduce_sum_algo(x, out_f32=out, algo=algo, stream=s)
        b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / k


x = gen.generate_tensor(gen.SEED_C3, 0, 1 << 30, gen.UNIFORM_PM1)
r20 = {a[0]: [] for a in arms}
for r in range(10):
    for name, algo, cfg in arms:
        setup(cfg)
        block(x, algo, 3)
        r20[name].append(block(x, algo, 20))
m0 = statistics.median(r20["mma_sync"])
print("2^30, 20 back-to-back, median of 10 interleaved rounds (min, max):")
for name, _, _ in arms:
    v = r20[name]
    print(f"  {name:14s} {statistics.median(v):7.1f} us ({min(v):.1f}, {max(v):.1f})  "
          f"{2 ** 31 / statistics.median(v) / 1e3:6.0f} GB/s  {statistics.median(v) / m0:.3f}x", flush=True)
sus = {a[0]: [] for a in arms}
for r in range(3):
    for name, algo, cfg in arms:
        setup(cfg)
        sus[name].append(block(x, algo, 200))
print("2^30 sustained (blocks of 200, 3 rounds): " + " | ".join(
    f"{n} {statistics.median(v):.1f}" for n, v in sus.items()), flush=True)
del x
for lg in (22, 24, 26, 28):
    xs = gen.generate_tensor(gen.SEED_C2, 0, 1 << lg, gen.UNIFORM_PM1)
    row = []
    for name, algo, cfg in arms:
        setup(cfg)
        t = statistics.median(graph_time(lambda: tcr.tcr_reduce_sum_algo(xs, out_f32=out, algo=algo),
                                         reps=100 if lg <= 24 else 20) for _ in range(3))
        row.append(f"{name} {t:7.2f}")
    print(f"2^{lg} warm: " + " | ".join(row), flush=True)
    del xs
for k, v in zip(bk, saved):
    tcr.tcr_set_config(k, v)
