"""A/B of libtcr builds on the batched entry (r02 rows-as-MMA-rows kernel):
tcr_reduce_sum_batched_ex(f16, MMA) for L in (64, 256, 1024, 2048) over 1 GiB,
rounds interleaved across the builds, each round = 50 back-to-back launches
between one event pair.  Usage: python scripts/ab_rows.py LIB [LIB ...]"""
import ctypes
import statistics
import sys

import torch

sys.path.insert(0, ".")
import tcr_inputs as gen  # noqa: E402

libs = sys.argv[1:]
fns = []
for p in libs:
    f = ctypes.CDLL(p).tcr_reduce_sum_batched_ex
    f.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_void_p,
                  ctypes.c_int, ctypes.c_void_p]
    f.restype = ctypes.c_int
    fns.append(f)
s = torch.cuda.Stream()
for L in (64, 256, 1024, 2048):
    S = (1 << 29) // L
    x = gen.generate_tensor(gen.SEED_C5, 0, L * S, gen.UNIFORM_PM1)
    out = torch.empty(S, dtype=torch.float32, device="cuda")
    res = {p: [] for p in libs}
    for r in range(6):
        for p, f in zip(libs, fns):
            for _ in range(3):
                assert f(x.data_ptr(), 0, S, L, out.data_ptr(), 1, s.cuda_stream) == 0
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(50):
                f(x.data_ptr(), 0, S, L, out.data_ptr(), 1, s.cuda_stream)
            b.record(s)
            torch.cuda.synchronize()
            res[p].append(a.elapsed_time(b) * 1e3 / 50)
    for p in libs:
        us = statistics.median(res[p])
        print(f"L={L:5d} {p:40s} {us:8.1f} us  {(2 * S * L + 4 * S) / (us * 1e-6) / 1e9:7.1f} GB/s", flush=True)
    del x
