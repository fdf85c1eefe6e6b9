"""Fixed-length batched reductions (SURVEY §8(d) C5 sweep): L = 256, 4096 at
2^20 segments and L = 65536 at 2^17 segments; CUDA-event time per launch
(median of 20 after 3 warm-up), effective GB/s = (2*S*L + 4*S) / t."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402

for L, S in ((256, 1 << 20), (1024, 1 << 20), (4096, 1 << 20), (65536, 1 << 17)):
    x = gen.generate_tensor(gen.SEED_C5, 0, L * S, gen.UNIFORM_PM1)
    out = torch.empty(S, dtype=torch.float32, device="cuda")
    for name, fn in (("mma", tcr.tcr_reduce_sum_batched), ("shuffle", tcr.tcr_reduce_sum_batched_shuffle)):
        ts = []
        for i in range(23):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn(x, L, out)
            b.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(a.elapsed_time(b))
        ms = statistics.median(ts)
        print(f"L={L:6d} S={S:8d} {name:8s} {ms*1e3:9.1f} us  {(2*S*L+4*S)/(ms*1e-3)/1e9:8.1f} GB/s", flush=True)
    del x
