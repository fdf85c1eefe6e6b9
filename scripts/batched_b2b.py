"""Fixed-length batched reductions, back-to-back launches (r02): 1 GiB of
binary16 per L (S = 2^29 / L rows), 3 warm-up then 50 launches between one
event pair on one stream; GB/s = (2 S L + 4 S) / t.  MMA path (rows-as-MMA-
rows kernel for L % 32 == 0 and L <= 2048, union-stream kernel otherwise)
and the shuffle path."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402

s = torch.cuda.Stream()
for L in (32, 64, 128, 256, 512, 1024, 2048, 4096, 65536):
    S = (1 << 29) // L
    x = gen.generate_tensor(gen.SEED_C5, 0, L * S, gen.UNIFORM_PM1)
    out = torch.empty(S, dtype=torch.float32, device="cuda")
    for algo in ("mma_sync", "shuffle"):
        with torch.cuda.stream(s):
            for _ in range(3):
                tcr.tcr_reduce_sum_batched_ex(x, L, out, algo=algo, stream=s)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(50):
                tcr.tcr_reduce_sum_batched_ex(x, L, out, algo=algo, stream=s)
            b.record(s)
        torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3 / 50
        print(f"L={L:6d} S={S:9d} {algo:8s} {us:9.1f} us  {(2 * S * L + 4 * S) / (us * 1e-6) / 1e9:8.1f} GB/s",
              flush=True)
    del x
