"""bps 4 vs 8 at 2^27..2^29 (graph-timed)."""
import statistics, sys
import torch
sys.path.insert(0, "."); sys.path.insert(0, "scripts")
import paper_1903_03640_b200 as tcr
import tcr_inputs as gen
from c2_compare_lib import graph_time
o = torch.empty(1, dtype=torch.float32, device="cuda")
for lg in (26, 27, 28, 29):
    n = 1 << lg
    x = gen.generate_tensor(gen.SEED_C3, 0, n, gen.UNIFORM_PM1)
    row = []
    for bps in (4, 8):
        tcr.tcr_set_config(tcr.TCR_CFG_BLOCKS_PER_SM, bps)
        # stream_grid caps at the resident wave below 2^28 unless unroll is forced; force U=4
        tcr.tcr_set_config(tcr.TCR_CFG_UNROLL, 4)
        t = statistics.median(graph_time(lambda: tcr.tcr_reduce_sum_algo(x, out_f32=o, algo="mma_sync"), 20) for _ in range(3))
        row.append(f"bps{bps}:{t:7.2f}")
    tcr.tcr_set_config(tcr.TCR_CFG_UNROLL, 0)
    t = statistics.median(graph_time(lambda: tcr.tcr_reduce_sum_algo(x, out_f32=o, algo="mma_sync"), 20) for _ in range(3))
    row.append(f"default(bps8,auto):{t:7.2f}")
    print(f"n=2^{lg}: " + " ".join(row), flush=True)
    del x
