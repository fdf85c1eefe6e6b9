"""The paper's question measured: time of the MMA-encoded reduction vs the
classic shuffle tree (and torch.sum, and the paper's algorithm taken
literally -- fp16 partials, one launch per level) across n = 2^10 .. 2^32, warm, CUDA
graph of back-to-back launches (graph_time), median of 3.  The paper's model
predicts S = T/T_tc = 6.4 at every n; on B200 both paths are bound by
latency (small n) or HBM (large n), so the measured ratio is ~1.
Writes gpurun_out/speedup_curve.json."""
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402
from c2_compare_lib import graph_time  # noqa: E402

rows = []
out = torch.empty(1, dtype=torch.float32, device="cuda")
for lg in range(10, 33, 2):
    n = 1 << lg
    x = gen.generate_tensor(gen.SEED_C2, 0, n, gen.UNIFORM_PM1)
    reps = 100 if lg <= 26 else 10
    t = {}
    for name, fn in (("default", lambda: tcr.tcr_reduce_sum_algo(x, out_f32=out, algo="default")),
                     ("mma_sync", lambda: tcr.tcr_reduce_sum_algo(x, out_f32=out, algo="mma_sync")),
                     ("tcgen05", lambda: tcr.tcr_reduce_sum_algo(x, out_f32=out, algo="tcgen05")),
                     ("shuffle", lambda: tcr.tcr_reduce_sum_algo(x, out_f32=out, algo="shuffle")),
                     ("torch.sum", lambda: torch.sum(x, dtype=torch.float32)),
                     ("paper_f16", lambda: tcr.tcr_reduce_sum_paper_f16(x, out))):
        t[name] = statistics.median(graph_time(fn, reps) for _ in range(3))
    row = {"log2n": lg, **{k + "_us": v for k, v in t.items()},
           "shuffle_over_mma": t["shuffle"] / t["mma_sync"],
           "mma_gbs": 2 * n / (t["mma_sync"] * 1e-6) / 1e9}
    rows.append(row)
    print(f"n=2^{lg:2d}: mma {t['mma_sync']:9.2f} us  tcgen05 {t['tcgen05']:9.2f}  shuffle "
          f"{t['shuffle']:9.2f}  torch.sum {t['torch.sum']:9.2f}  paper_f16 {t['paper_f16']:9.2f}  shuffle/mma "
          f"{row['shuffle_over_mma']:.3f}  ({row['mma_gbs']:.0f} GB/s)", flush=True)
    del x
with open("gpurun_out/speedup_curve.json", "w") as f:
    json.dump({"paper_model_S": 6.4, "rows": rows}, f, indent=1)
