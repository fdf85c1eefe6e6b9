python - <<'PY'
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
for lg in (26, 27, 29, 31):
    n = 1 << lg
    for dt in ("f16", "e4m3"):
        if dt == "f16" and lg == 31: continue
        x = gen.generate_tensor(gen.SEED_C3, 0, n, gen.UNIFORM_PM1) if dt == "f16" else gen.generate_tensor_fp8(gen.SEED_C3, 0, n, gen.UNIFORM_PM1, gen.FP8_E4M3)
        es = 2 if dt == "f16" else 1
        res = {}
        for r in range(5):
            for name, eb in (("ldg", 0), ("bulk", 2)):
                tcr.tcr_set_config(tcr.TCR_CFG_EXACT_BULK, eb)
                f = lambda: tcr.tcr_reduce_sum_exact_ex(x, out_f32=out, stream=s)
                if r == 0: b2b(f, 5)
                res.setdefault(name, []).append(b2b(f))
        tcr.tcr_set_config(tcr.TCR_CFG_EXACT_BULK, 1)
        print(f"{dt} 2^{lg}: " + " | ".join(f"exact {k} {statistics.median(v):9.2f} us {es*n/statistics.median(v)/1e3:6.0f} GB/s" for k, v in res.items()), flush=True)
        del x; torch.cuda.empty_cache()
PY
