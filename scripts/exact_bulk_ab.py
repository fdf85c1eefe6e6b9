"""r02 §18: the exact reduction, LDG kernel vs the TMA-fed kernel with the dynamic tail vs the tcgen05 default, back to back (20 launches, median of 6 interleaved rounds)."""
import statistics, sys, torch
sys.path.insert(0, ".")
import paper_1903_03640_b200 as tcr, tcr_inputs as gen
out = torch.empty(1, dtype=torch.float32, device="cuda"); s = torch.cuda.Stream()
def b2b(f, k=20):
    with torch.cuda.stream(s):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(k): f()
        b.record(s)
    torch.cuda.synchronize(); return a.elapsed_time(b) * 1e3 / k
for lg in (28, 29, 30, 32):
    n = 1 << lg
    x = gen.generate_tensor(gen.SEED_C3, 0, n, gen.UNIFORM_PM1)
    res = {}
    arms = (("exact ldg", 0, None), ("exact bulk", 2, None), ("tcgen05", None, "tcgen05"))
    for r in range(6):
        for name, eb, algo in arms:
            if eb is not None:
                tcr.tcr_set_config(tcr.TCR_CFG_EXACT_BULK, eb)
                f = lambda: tcr.tcr_reduce_sum_exact(x, out_f32=out, stream=s)
            else:
                f = lambda: tcr.tcr_reduce_sum_algo(x, out_f32=out, algo="tcgen05", stream=s)
            if r == 0: b2b(f, 5)
            res.setdefault(name, []).append(b2b(f))
    tcr.tcr_set_config(tcr.TCR_CFG_EXACT_BULK, 1)
    print(f"2^{lg}: " + " | ".join(f"{k} {statistics.median(v):9.2f} us {2*n/statistics.median(v)/1e3:6.0f} GB/s" for k, v in res.items()), flush=True)
    del x; torch.cuda.empty_cache()
