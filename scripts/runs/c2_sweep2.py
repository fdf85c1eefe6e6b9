"""Small-n latency sweep, 5 trials per point (median): CUDA graph of 100 launches."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402
from c2_compare_lib import graph_time  # noqa: E402

for n in (1 << 20, 1 << 22, 1 << 23, 1 << 24, 1 << 25):
    x = gen.generate_tensor(gen.SEED_C2, 0, n, gen.UNIFORM_PM1)
    out = torch.empty(1, dtype=torch.float32, device="cuda")
    row = []
    for u in (0, 4, 8, 16):
        for b in ((1, 2, 3, 4) if u else (8,)):
            tcr.tcr_set_config(tcr.TCR_CFG_UNROLL, u)
            tcr.tcr_set_config(tcr.TCR_CFG_BLOCKS_PER_SM, b)
            t = statistics.median(graph_time(lambda: tcr.tcr_reduce_sum_algo(x, out_f32=out, algo="mma_sync"))
                                  for _ in range(5))
            row.append(f"u{u}b{b}:{t:5.2f}")
    print(f"n=2^{n.bit_length()-1}: " + " ".join(row), flush=True)
