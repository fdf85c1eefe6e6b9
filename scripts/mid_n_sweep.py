"""mma.sync streaming kernel between C2 and C3 (2^25..2^28): unroll x
CTAs/SM, graph-timed warm (the auto rule: unroll 16 below 2^26 elements, 4
above; one resident wave below 2^28)."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402
from c2_compare_lib import graph_time  # noqa: E402

out = torch.empty(1, dtype=torch.float32, device="cuda")
for lg in (25, 26, 27, 28):
    x = gen.generate_tensor(gen.SEED_C2, 0, 1 << lg, gen.UNIFORM_PM1)
    row = []
    for u in (0, 4, 8, 16):
        for b in (4, 8):
            tcr.tcr_set_config(tcr.TCR_CFG_UNROLL, u)
            tcr.tcr_set_config(tcr.TCR_CFG_BLOCKS_PER_SM, b)
            t = statistics.median(graph_time(lambda: tcr.tcr_reduce_sum_algo(x, out_f32=out, algo="mma_sync"),
                                             reps=20) for _ in range(3))
            row.append(f"u{u}b{b} {t:6.2f}")
    tcr.tcr_set_config(tcr.TCR_CFG_UNROLL, 0)
    tcr.tcr_set_config(tcr.TCR_CFG_BLOCKS_PER_SM, 8)
    print(f"2^{lg}: " + " | ".join(row), flush=True)
    del x
