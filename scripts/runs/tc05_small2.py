import statistics, sys
import torch
sys.path.insert(0, "."); sys.path.insert(0, "scripts")
import paper_1903_03640_b200 as tcr
import tcr_inputs as gen
from c2_compare_lib import graph_time
o = torch.empty(1, dtype=torch.float32, device="cuda")
for lg in (16, 20, 22, 24, 26, 28):
    n = 1 << lg
    x = gen.generate_tensor(gen.SEED_C2, 0, n, gen.UNIFORM_PM1)
    row = []
    for ctas in (1, 2, 3):
        for kb in (16, 8):
            tcr.tcr_set_config(tcr.TCR_CFG_TC05_CTAS_PER_SM, ctas)
            tcr.tcr_set_config(tcr.TCR_CFG_TC05_STAGE_KB, kb)
            t = statistics.median(graph_time(lambda: tcr.tcr_reduce_sum_algo(x, out_f32=o, algo="tcgen05"), 50 if lg < 28 else 10) for _ in range(3))
            row.append(f"c{ctas}k{kb}:{t:6.2f}")
    print(f"n=2^{lg}: " + " ".join(row), flush=True)
