"""A/B experiment (needs build/ab/libtcr_w4.so: the streaming kernel rebuilt with 4-warp CTAs): 8-warp CTAs at bps 8 vs 4-warp CTAs at bps 8/16/24.  Result (r01): 295.5 vs 297.2 / 296.3 / 298.9 us -- no gain."""
import ctypes, statistics, sys
import torch
sys.path.insert(0, ".")
import tcr_inputs as gen

def load(path, bps):
    lib = ctypes.CDLL(path)
    lib.tcr_set_config(1, bps)
    f = lib.tcr_reduce_sum_ex
    f.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    return lib, f

n = 1 << 30
x = gen.generate_tensor(gen.SEED_C3, 0, n, gen.UNIFORM_PM1)
out = torch.empty(1, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()
cfgs = [("w8 bps8", "paper_1903_03640_b200/libtcr.so", 8)]
for b in (8, 16, 24):
    cfgs.append((f"w4 bps{b}", "build/ab/libtcr_w4.so", b))
libs = {}
res = {}
for rnd in range(4):
    for name, path, bps in cfgs:
        if path not in libs:
            libs[path] = load(path, bps)
        lib, f = libs[path]
        lib.tcr_set_config(1, bps)
        for _ in range(3):
            f(x.data_ptr(), n, 0, out.data_ptr(), None, 1, s.cuda_stream)
        a, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(50):
            f(x.data_ptr(), n, 0, out.data_ptr(), None, 1, s.cuda_stream)
        b2.record(s)
        torch.cuda.synchronize()
        res.setdefault(name, []).append(a.elapsed_time(b2) * 1e3 / 50)
for k, ts in res.items():
    us = statistics.median(ts)
    print(f"{k}: {us:7.2f} us  {2 * n / us / 1e3:7.1f} GB/s  {[round(t, 1) for t in ts]}")
