import statistics, sys
import torch
sys.path.insert(0, "."); sys.path.insert(0, "scripts")
import paper_1903_03640_b200 as tcr
import tcr_inputs as gen
from c2_compare_lib import graph_time
for lg in (16, 20, 22, 24, 26):
    n = 1 << lg
    x = gen.generate_tensor(gen.SEED_C2, 0, n, gen.UNIFORM_PM1)
    o = torch.empty(1, dtype=torch.float32, device="cuda")
    te = statistics.median(graph_time(lambda: tcr.tcr_reduce_sum_exact(x, out_f32=o)) for _ in range(3))
    tm = statistics.median(graph_time(lambda: tcr.tcr_reduce_sum_algo(x, out_f32=o, algo="mma_sync")) for _ in range(3))
    print(f"n=2^{lg}: exact {te:6.2f} us  mma_sync {tm:6.2f} us")
