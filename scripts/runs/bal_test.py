"""Balanced-batch experiment (reverted; needs the TCR_CFG_BALANCE build of the streaming kernel): parity + determinism, then A/B timing."""
import statistics, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle
import paper_1903_03640_b200 as tcr
import tcr_inputs as gen

o = torch.empty(1, dtype=torch.float32, device="cuda")
tcr.tcr_set_config(tcr.TCR_CFG_BALANCE, 1)
for n, dist, off in (((1 << 26) + 77, gen.UNIFORM_01, 1), ((1 << 27) + 5, gen.WIDE, 3), (1 << 26, gen.SMALLINT, 0)):
    bits = gen.generate(7, 0, n, dist)
    es = oracle.exact_sum_fp16(bits, threads=16)
    buf = torch.empty(n + 16, dtype=torch.int16, device="cuda")
    x = buf[off:off + n]
    x.copy_(torch.from_numpy(bits.view(np.int16)))
    x = x.view(torch.float16)
    for algo in ("mma_sync", "shuffle"):
        tcr.tcr_reduce_sum_algo(x, out_f32=o, algo=algo); torch.cuda.synchronize()
        g = float(o.item())
        tcr.tcr_reduce_sum_algo(x, out_f32=o, algo=algo); torch.cuda.synchronize()
        assert g == float(o.item()), "nondeterministic"
        assert oracle.within_tolerance(g, es), (n, algo, g, es.f64())
        if dist == gen.SMALLINT:
            assert g == es.f32()
    del buf, x
print("parity ok")
n = 1 << 30
x = gen.generate_tensor(gen.SEED_C3, 0, n, gen.UNIFORM_PM1)
s = torch.cuda.current_stream()
res = {}
for rnd in range(4):
    for bal, bps in ((0, 8), (1, 8), (1, 4), (1, 12)):
        tcr.tcr_set_config(tcr.TCR_CFG_BALANCE, bal)
        tcr.tcr_set_config(tcr.TCR_CFG_BLOCKS_PER_SM, bps)
        for _ in range(3):
            tcr.tcr_reduce_sum_algo(x, out_f32=o, algo="mma_sync")
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(50):
            tcr.tcr_reduce_sum_algo(x, out_f32=o, algo="mma_sync")
        b.record(s)
        torch.cuda.synchronize()
        res.setdefault((bal, bps), []).append(a.elapsed_time(b) * 1e3 / 50)
for k, ts in res.items():
    us = statistics.median(ts)
    print(f"balance {k[0]} bps {k[1]:2d}: {us:7.2f} us  {2 * n / us / 1e3:7.1f} GB/s   all {[round(t,1) for t in ts]}")
