"""The TMA-fed mma.sync path ("bulk": cp.async.bulk -> SMEM ring -> ld.shared
-> mma.sync) vs the LDG-fed default, r02: ring shapes at 2^30 and 2^32,
back-to-back launches (2^30: 20, 2^32: 5), mma.sync and tcgen05 as
references.  Config = (stages, KiB, CTAs/SM)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402

keys = (tcr.TCR_CFG_BULK_STAGES, tcr.TCR_CFG_BULK_STAGE_KB, tcr.TCR_CFG_BULK_CTAS_PER_SM)
saved = [tcr.tcr_get_config(k) for k in keys]
out = torch.empty(1, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()


def b2b(x, algo, k):
    with torch.cuda.stream(s):
        for _ in range(2):
            tcr.tcr_reduce_sum_algo(x, out_f32=out, algo=algo, stream=s)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(k):
            tcr.tcr_reduce_sum_algo(x, out_f32=out, algo=algo, stream=s)
        b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / k


for lg, k in ((30, 20), (32, 5)):
    x = gen.generate_tensor(gen.SEED_C3, 0, 1 << lg, gen.UNIFORM_PM1)
    gb = lambda us: 2 * (1 << lg) / us / 1e3  # noqa: E731
    row = []
    for algo in ("mma_sync", "tcgen05"):
        t = b2b(x, algo, k)
        row.append(f"{algo} {t:8.1f} us {gb(t):5.0f}")
    for cfg in ((6, 16, 2), (3, 32, 2), (4, 32, 1), (3, 64, 1), (2, 64, 1), (6, 32, 1), (12, 16, 1)):
        for kk, v in zip(keys, cfg):
            tcr.tcr_set_config(kk, v)
        t = b2b(x, "bulk", k)
        row.append(f"bulk {cfg[0]}x{cfg[1]}c{cfg[2]} {t:8.1f} us {gb(t):5.0f}")
    print(f"n=2^{lg}: " + " | ".join(row), flush=True)
    del x
for kk, v in zip(keys, saved):
    tcr.tcr_set_config(kk, v)
