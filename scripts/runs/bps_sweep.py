"""Back-to-back device time per launch at 2^30 vs CTAs per SM (grid waves)."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402

n = 1 << 30
x = gen.generate_tensor(gen.SEED_C3, 0, n, gen.UNIFORM_PM1)
out = torch.empty(1, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()
res = {}
for rnd in range(3):
    for bps in (4, 6, 8, 12, 16, 24, 32):
        tcr.tcr_set_config(tcr.TCR_CFG_BLOCKS_PER_SM, bps)
        for _ in range(3):
            tcr.tcr_reduce_sum_algo(x, out_f32=out, algo="mma_sync")
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(50):
            tcr.tcr_reduce_sum_algo(x, out_f32=out, algo="mma_sync")
        b.record(s)
        torch.cuda.synchronize()
        res.setdefault(bps, []).append(a.elapsed_time(b) * 1e3 / 50)
for bps, ts in res.items():
    us = statistics.median(ts)
    print(f"bps {bps:2d}: {us:7.2f} us  {2 * n / us / 1e3:7.1f} GB/s")
