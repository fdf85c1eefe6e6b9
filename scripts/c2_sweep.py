"""Small-n (C2, n = 2^24) latency vs launch configuration of the mma.sync
kernel: CUDA graph of 100 back-to-back launches (warm) per (unroll, CTAs/SM)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402

sys.path.insert(0, "scripts")
from c2_compare_lib import graph_time  # noqa: E402

for n in (1 << 20, 1 << 22, 1 << 24, 1 << 26):
    x = gen.generate_tensor(gen.SEED_C2, 0, n, gen.UNIFORM_PM1)
    out = torch.empty(1, dtype=torch.float32, device="cuda")
    row = []
    for u in (4, 8):
        for b in (1, 2, 4, 8):
            tcr.tcr_set_config(tcr.TCR_CFG_UNROLL, u)
            tcr.tcr_set_config(tcr.TCR_CFG_BLOCKS_PER_SM, b)
            us = graph_time(lambda: tcr.tcr_reduce_sum_algo(x, out_f32=out, algo="mma_sync"))
            row.append(f"u{u}b{b}:{us:6.2f}")
    print(f"n=2^{n.bit_length()-1}: " + " ".join(row), flush=True)
