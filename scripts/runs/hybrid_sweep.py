"""tcgen05 hybrid experiment (reverted; needed a TCR_CFG_TC05_LDG_PERMILLE build): epilogue warps also streaming part of the input with LDG + mma.sync.  r01 result: every share was slower (0: 304.0, 5 %: 322.1, 30 %: 386.3 us; mma.sync 298.5)."""
back-to-back timing vs the share, against the default mma.sync path."""
import statistics, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle
import paper_1903_03640_b200 as tcr
import tcr_inputs as gen
o = torch.empty(1, dtype=torch.float32, device="cuda")
# parity
bits = gen.generate(3, 0, (1 << 24) + 12345, gen.UNIFORM_01)
es = oracle.exact_sum_fp16(bits, threads=8)
xs = torch.from_numpy(bits.view(np.int16)).cuda().view(torch.float16)
for pm in (0, 50, 150, 300, 600):
    tcr.tcr_set_config(tcr.TCR_CFG_TC05_LDG_PERMILLE, pm)
    tcr.tcr_reduce_sum_algo(xs, out_f32=o, algo="tcgen05"); torch.cuda.synchronize()
    g = float(o.item())
    tcr.tcr_reduce_sum_algo(xs, out_f32=o, algo="tcgen05"); torch.cuda.synchronize()
    assert g == float(o.item()) and oracle.within_tolerance(g, es), (pm, g, es.f64())
print("parity ok", flush=True)
n = 1 << 30
x = gen.generate_tensor(gen.SEED_C3, 0, n, gen.UNIFORM_PM1)
s = torch.cuda.current_stream()
res = {}
for rnd in range(3):
    for name, algo, pm in [("mma_sync", "mma_sync", 0)] + [(f"tc05 ldg{pm}", "tcgen05", pm) for pm in (0, 50, 100, 150, 200, 300)]:
        tcr.tcr_set_config(tcr.TCR_CFG_TC05_LDG_PERMILLE, pm)
        for _ in range(3):
            tcr.tcr_reduce_sum_algo(x, out_f32=o, algo=algo)
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(40):
            tcr.tcr_reduce_sum_algo(x, out_f32=o, algo=algo)
        e.record(s)
        torch.cuda.synchronize()
        res.setdefault(name, []).append(a.elapsed_time(e) * 1e3 / 40)
for k, ts in res.items():
    us = statistics.median(ts)
    print(f"{k:14s}: {us:7.2f} us  {2 * n / us / 1e3:7.1f} GB/s", flush=True)
