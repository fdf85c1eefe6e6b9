"""tcgen05 with the library's automatic small-input ring shapes vs mma.sync, warm CUDA graphs, 2^20..2^27 (r02)."""
import statistics, sys, torch
sys.path.insert(0, "."); sys.path.insert(0, "scripts")
import paper_1903_03640_b200 as tcr, tcr_inputs as gen
from c2_compare_lib import graph_time
out = torch.empty(1, dtype=torch.float32, device="cuda")
for lg in range(20, 28):
    x = gen.generate_tensor(gen.SEED_C2, 0, 1 << lg, gen.UNIFORM_PM1)
    m = statistics.median(graph_time(lambda: tcr.tcr_reduce_sum_algo(x, out_f32=out, algo="mma_sync")) for _ in range(3))
    t = statistics.median(graph_time(lambda: tcr.tcr_reduce_sum_algo(x, out_f32=out, algo="tcgen05")) for _ in range(3))
    print(f"n=2^{lg}: mma.sync {m:6.2f} us | tcgen05 (library auto shape) {t:6.2f} us ({t/m:.2f} x)", flush=True)
