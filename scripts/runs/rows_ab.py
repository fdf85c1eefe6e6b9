"""A/B of the batched rows kernel (fixed L, 2^20 rows) between libtcr builds (back-to-back launches).  Used to reject a batched-DMMA row collapse (r01): L=256 82.0 vs 84.5 us."""
import ctypes, statistics, sys
import torch
sys.path.insert(0, ".")
import tcr_inputs as gen
libs = sys.argv[1:]
fns = []
for p in libs:
    f = ctypes.CDLL(p).tcr_reduce_sum_batched
    f.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p]
    fns.append(f)
s = torch.cuda.current_stream()
for L, S in ((256, 1 << 20), (512, 1 << 20), (1024, 1 << 20), (2048, 1 << 19)):
    x = gen.generate_tensor(L, 0, L * S, gen.UNIFORM_PM1)
    out = torch.empty(S, dtype=torch.float32, device="cuda")
    row = []
    for p, f in zip(libs, fns):
        for _ in range(3):
            f(x.data_ptr(), S, L, out.data_ptr(), s.cuda_stream)
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(20):
                f(x.data_ptr(), S, L, out.data_ptr(), s.cuda_stream)
            b.record(s)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3 / 20)
        us = statistics.median(ts)
        row.append(f"{p.split('/')[-1]}: {us:7.2f} us {2 * L * S / us / 1e3:6.0f} GB/s")
    print(f"L={L} S={S}: " + " | ".join(row), flush=True)
    del x
