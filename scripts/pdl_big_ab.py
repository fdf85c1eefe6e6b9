"""PDL on / off for the large-n kernels (r02): 2^31..2^33, 10 back-to-back
launches between one event pair (median of 3 batches), mma.sync and tcgen05."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402

out = torch.empty(1, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()


def b2b(x, algo, k=10):
    ts = []
    for _ in range(3):
        with torch.cuda.stream(s):
            tcr.tcr_reduce_sum_algo(x, out_f32=out, algo=algo, stream=s)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(k):
                tcr.tcr_reduce_sum_algo(x, out_f32=out, algo=algo, stream=s)
            b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / k)
    return statistics.median(ts)


for lg in (31, 32, 33):
    x = gen.generate_tensor(gen.SEED_C4, 0, 1 << lg, gen.UNIFORM_PM1)
    row = []
    for algo in ("mma_sync", "tcgen05"):
        for pdl in (1, 0):
            tcr.tcr_set_config(tcr.TCR_CFG_PDL, pdl)
            t = b2b(x, algo)
            row.append(f"{algo}/pdl{pdl} {t:8.1f} us {2 * (1 << lg) / t / 1e3:5.0f} GB/s")
    tcr.tcr_set_config(tcr.TCR_CFG_PDL, 1)
    print(f"2^{lg}: " + " | ".join(row), flush=True)
    del x
