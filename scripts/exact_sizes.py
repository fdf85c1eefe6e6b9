import sys, statistics, torch
sys.path.insert(0, ".")
import paper_1903_03640_b200 as tcr, tcr_inputs as gen
out = torch.empty(1, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
def b2b(f, k=20):
    with torch.cuda.stream(s):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(k): f()
        b.record(s)
    torch.cuda.synchronize(); return a.elapsed_time(b)*1e3/k
for lg in (28, 30, 32):
    n = 1 << lg
    x = gen.generate_tensor(gen.SEED_C3, 0, n, gen.UNIFORM_PM1)
    fe = lambda: tcr.tcr_reduce_sum_exact(x, out_f32=out, stream=s)
    ft = lambda: tcr.tcr_reduce_sum_algo(x, out_f32=out, algo="tcgen05", stream=s)
    for f in (fe, ft): b2b(f, 10)
    te = statistics.median(b2b(fe) for _ in range(5)); tt = statistics.median(b2b(ft) for _ in range(5))
    print(f"2^{lg}: exact {te:9.2f} us {2*n/te/1e3:6.0f} GB/s | tcgen05 dyn {tt:9.2f} us {2*n/tt/1e3:6.0f} GB/s", flush=True)
    del x; torch.cuda.empty_cache()
