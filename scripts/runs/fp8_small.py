import statistics, sys
import torch
sys.path.insert(0, "."); sys.path.insert(0, "scripts")
import paper_1903_03640_b200 as tcr
import tcr_inputs as gen
from c2_compare_lib import graph_time
o = torch.empty(1, dtype=torch.float32, device="cuda")
for lg in (16, 20, 22, 24, 26, 27, 28, 30):
    n = 1 << lg
    x = gen.generate_tensor_fp8(gen.SEED_C2, 0, n, gen.UNIFORM_PM1, gen.FP8_E4M3)
    t = {a: statistics.median(graph_time(lambda: tcr.tcr_reduce_sum_ex(x, out_f32=o, algo=a), 100 if lg < 28 else 10) for _ in range(3))
         for a in ("tcgen05", "mma_sync", "shuffle")}
    print(f"fp8 n=2^{lg}: " + "  ".join(f"{k} {v:8.2f}" for k, v in t.items()), flush=True)
