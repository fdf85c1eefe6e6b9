"""tcgen05 (tight issue loop) below 256 MiB: CTAs per SM and ring shape vs
latency, graph-timed (100 launches, median of 3); mma.sync as reference.
Config = (stages, KiB, slots, chain, CTAs/SM); one round per stage requires
slots * chain = KiB / 4."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402
from c2_compare_lib import graph_time  # noqa: E402

keys = (tcr.TCR_CFG_TC05_STAGES, tcr.TCR_CFG_TC05_STAGE_KB, tcr.TCR_CFG_TC05_SLOTS,
        tcr.TCR_CFG_TC05_CHAIN, tcr.TCR_CFG_TC05_CTAS_PER_SM)
saved = [tcr.tcr_get_config(k) for k in keys]
cfgs = [(2, 32, 4, 2, 3), (2, 16, 4, 1, 4), (3, 16, 4, 1, 4), (4, 16, 4, 1, 3), (3, 32, 4, 2, 2),
        (2, 16, 4, 1, 3), (6, 16, 4, 1, 2), (4, 32, 4, 2, 1)]
out = torch.empty(1, dtype=torch.float32, device="cuda")
for lg in [int(a) for a in sys.argv[1:]] or (20, 22, 24, 26):
    x = gen.generate_tensor(gen.SEED_C2, 0, 1 << lg, gen.UNIFORM_PM1)
    m = statistics.median(graph_time(lambda: tcr.tcr_reduce_sum_algo(x, out_f32=out, algo="mma_sync"))
                          for _ in range(3))
    row = [f"mma {m:5.2f}"]
    for c in cfgs:
        for k, v in zip(keys, c):
            tcr.tcr_set_config(k, v)
        t = statistics.median(graph_time(lambda: tcr.tcr_reduce_sum_algo(x, out_f32=out, algo="tcgen05"))
                              for _ in range(3))
        row.append(f"{c[0]}x{c[1]}c{c[4]} {t:5.2f} ({t / m:.2f})")
    print(f"n=2^{lg}: " + " | ".join(row), flush=True)
for k, v in zip(keys, saved):
    tcr.tcr_set_config(k, v)
