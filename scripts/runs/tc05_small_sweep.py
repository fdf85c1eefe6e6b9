"""tcgen05 small-n latency vs knobs (graph-timed, median of 3)."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402
from c2_compare_lib import graph_time  # noqa: E402

for n in (1 << 22, 1 << 24, 1 << 26):
    x = gen.generate_tensor(gen.SEED_C2, 0, n, gen.UNIFORM_PM1)
    out = torch.empty(1, dtype=torch.float32, device="cuda")
    row = []
    for stages, kb, ctas in ((4, 16, 3), (4, 8, 3), (4, 4, 3), (8, 4, 3), (4, 4, 4), (2, 16, 3), (4, 8, 4), (6, 4, 4)):
        tcr.tcr_set_config(tcr.TCR_CFG_TC05_STAGES, stages)
        tcr.tcr_set_config(tcr.TCR_CFG_TC05_STAGE_KB, kb)
        tcr.tcr_set_config(tcr.TCR_CFG_TC05_CTAS_PER_SM, ctas)
        t = statistics.median(graph_time(lambda: tcr.tcr_reduce_sum_algo(x, out_f32=out, algo="tcgen05"))
                              for _ in range(3))
        row.append(f"s{stages}k{kb}c{ctas}:{t:6.2f}")
    print(f"n=2^{n.bit_length()-1}: " + " ".join(row), flush=True)
