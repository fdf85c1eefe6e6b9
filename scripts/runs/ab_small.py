"""Graph-timed A/B of libtcr builds at small n (tcr_reduce_sum_ex, mma_sync)."""
import ctypes, statistics, sys
import torch
sys.path.insert(0, "."); sys.path.insert(0, "scripts")
import tcr_inputs as gen
from c2_compare_lib import graph_time
libs = sys.argv[1:]
fns = []
for p in libs:
    f = ctypes.CDLL(p).tcr_reduce_sum_ex
    f.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    fns.append(f)
o = torch.empty(1, dtype=torch.float32, device="cuda")
for lg in (14, 15, 16, 17, 18, 19, 20):
    n = 1 << lg
    x = gen.generate_tensor(gen.SEED_C2, 0, n, gen.UNIFORM_PM1)
    row = []
    for p, f in zip(libs, fns):
        t = statistics.median(graph_time(lambda: f(x.data_ptr(), n, 0, o.data_ptr(), None, 1, torch.cuda.current_stream().cuda_stream)) for _ in range(5))
        row.append(f"{p.split('/')[-1]}:{t:5.2f}")
    print(f"n=2^{lg}: " + "  ".join(row), flush=True)
