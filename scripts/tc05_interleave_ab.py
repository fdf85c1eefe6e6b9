"""tcgen05 chunk-to-CTA mapping (r02): contiguous runs (interleave 0) vs chunks
b, b+G, ... (interleave 1), one CTA per SM -- isolated launches (an event pair
around each, 30 launches, median) and back-to-back (20 launches per event
pair, median of 5), at 2^30 and 2^33; mma.sync as reference."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402

out = torch.empty(1, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()


def isolated(x, algo):
    ts = []
    for _ in range(30):
        with torch.cuda.stream(s):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(200000)
            a.record(s)
            tcr.tcr_reduce_sum_algo(x, out_f32=out, algo=algo, stream=s)
            b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts[5:])


def b2b(x, algo, k=20):
    ts = []
    for _ in range(5):
        with torch.cuda.stream(s):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(k):
                tcr.tcr_reduce_sum_algo(x, out_f32=out, algo=algo, stream=s)
            b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / k)
    return statistics.median(ts)


for lg in (30, 33):
    x = gen.generate_tensor(gen.SEED_C4, 0, 1 << lg, gen.UNIFORM_PM1)
    k = 20 if lg == 30 else 4
    row = [f"mma iso {isolated(x, 'mma_sync'):8.1f} b2b {b2b(x, 'mma_sync', k):8.1f}"]
    for il in (0, 1):
        tcr.tcr_set_config(tcr.TCR_CFG_TC05_INTERLEAVE, il)
        row.append(f"tc05 il{il} iso {isolated(x, 'tcgen05'):8.1f} b2b {b2b(x, 'tcgen05', k):8.1f}")
    tcr.tcr_set_config(tcr.TCR_CFG_TC05_INTERLEAVE, 0)
    print(f"2^{lg}: " + " | ".join(row), flush=True)
    del x
