"""A/B device timing of two builds of libtcr on the same box and tensor:
tcr_reduce_sum_ex (fp16, algo given) at n = 2^30, rounds interleaved A, B,
A, B, ... each round = CUDA events around 100 back-to-back launches.
Usage: python scripts/ab_lib.py LIB_A LIB_B [algo=1] [rounds=10]
algo = "c5": tcr_reduce_sum_segmented on the C5 workload (2^20 log-uniform
segments) instead, 10 launches per round."""
import ctypes
import statistics
import sys

import torch

sys.path.insert(0, ".")
import tcr_inputs as gen  # noqa: E402


def load(path):
    lib = ctypes.CDLL(path)
    f = lib.tcr_reduce_sum_ex
    f.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p,
                  ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    f.restype = ctypes.c_int
    return f


def main_c5(a, b, rounds):
    S = 1 << 20
    lens = gen.loguniform_lengths(gen.SEED_C5, S)
    off = gen.offsets_from_lengths(lens)
    n = int(off[-1])
    x = gen.generate_tensor(gen.SEED_C5, 0, n, gen.UNIFORM_PM1)
    toff = torch.from_numpy(off).cuda()
    out = torch.empty(S, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream()
    fns = {}
    for k, path in (("A", a), ("B", b)):
        f = ctypes.CDLL(path).tcr_reduce_sum_segmented
        f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                      ctypes.c_void_p]
        f.restype = ctypes.c_int
        fns[k] = f
    res = {"A": [], "B": []}
    for f in fns.values():
        for _ in range(3):
            assert f(x.data_ptr(), toff.data_ptr(), S, out.data_ptr(), s.cuda_stream) == 0
    torch.cuda.synchronize()
    for _ in range(rounds):
        for k, f in fns.items():
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(10):
                f(x.data_ptr(), toff.data_ptr(), S, out.data_ptr(), s.cuda_stream)
            e1.record(s)
            torch.cuda.synchronize()
            res[k].append(e0.elapsed_time(e1) * 100)  # us per launch
    for k in res:
        med = statistics.median(res[k])
        print(f"c5 {k} {a if k == 'A' else b}: median {med:.1f} us  {2 * n / med / 1e3:.1f} GB/s")


def main_exact(a, b, rounds):
    n = 1 << 30
    x = gen.generate_tensor(gen.SEED_C3, 0, n, gen.UNIFORM_PM1)
    out = torch.empty(1, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream()
    fns = {}
    for k, path in (("A", a), ("B", b)):
        f = ctypes.CDLL(path).tcr_reduce_sum_exact
        f.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p,
                      ctypes.c_void_p, ctypes.c_void_p]
        f.restype = ctypes.c_int
        fns[k] = f
    res = {"A": [], "B": []}
    for f in fns.values():
        for _ in range(5):
            assert f(x.data_ptr(), n, None, out.data_ptr(), None, s.cuda_stream) == 0
    torch.cuda.synchronize()
    for _ in range(rounds):
        for k, f in fns.items():
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(100):
                f(x.data_ptr(), n, None, out.data_ptr(), None, s.cuda_stream)
            e1.record(s)
            torch.cuda.synchronize()
            res[k].append(e0.elapsed_time(e1) * 10)
    for k in res:
        med = statistics.median(res[k])
        print(f"exact {k} {a if k == 'A' else b}: median {med:.2f} us  {2 * n / med / 1e3:.1f} GB/s")


def main():
    a, b = sys.argv[1], sys.argv[2]
    if len(sys.argv) > 3 and sys.argv[3] == "exact":
        return main_exact(a, b, int(sys.argv[4]) if len(sys.argv) > 4 else 10)
    if len(sys.argv) > 3 and sys.argv[3] == "c5":
        return main_c5(a, b, int(sys.argv[4]) if len(sys.argv) > 4 else 10)
    algo = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 10
    n = 1 << 30
    x = gen.generate_tensor(gen.SEED_C3, 0, n, gen.UNIFORM_PM1)
    out = torch.empty(1, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream()
    fns = {"A": load(a), "B": load(b)}
    res = {"A": [], "B": []}
    for k, f in fns.items():  # warm-up
        for _ in range(20):
            assert f(x.data_ptr(), n, 0, out.data_ptr(), None, algo, s.cuda_stream) == 0
    torch.cuda.synchronize()
    for _ in range(rounds):
        for k, f in fns.items():
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(100):
                f(x.data_ptr(), n, 0, out.data_ptr(), None, algo, s.cuda_stream)
            e1.record(s)
            torch.cuda.synchronize()
            res[k].append(e0.elapsed_time(e1) * 10)  # us per launch
    for k in res:
        med = statistics.median(res[k])
        print(f"{k} {sys.argv[1 if k == 'A' else 2]}: median {med:.2f} us  "
              f"{2 * n / med / 1e3:.1f} GB/s  (min {min(res[k]):.2f}, max {max(res[k]):.2f})")


if __name__ == "__main__":
    main()
