"""Re-tune the default streaming knobs at 2^30 (back-to-back launches, interleaved rounds)."""
import statistics, sys
import torch
sys.path.insert(0, ".")
import paper_1903_03640_b200 as tcr
import tcr_inputs as gen
n = 1 << 30
x = gen.generate_tensor(gen.SEED_C3, 0, n, gen.UNIFORM_PM1)
o = torch.empty(1, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()
cfgs = [(u, b, k) for u in (4, 8) for b in (7, 8, 9, 10, 12) for k in (4,)] + [(4, 8, 8), (8, 8, 8)]
res = {}
for rnd in range(3):
    for u, b, k in cfgs:
        tcr.tcr_set_config(tcr.TCR_CFG_UNROLL, u)
        tcr.tcr_set_config(tcr.TCR_CFG_BLOCKS_PER_SM, b)
        tcr.tcr_set_config(tcr.TCR_CFG_CHAIN, k)
        for _ in range(3):
            tcr.tcr_reduce_sum_algo(x, out_f32=o, algo="mma_sync")
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(40):
            tcr.tcr_reduce_sum_algo(x, out_f32=o, algo="mma_sync")
        e.record(s)
        torch.cuda.synchronize()
        res.setdefault((u, b, k), []).append(a.elapsed_time(e) * 1e3 / 40)
for key, ts in sorted(res.items(), key=lambda kv: statistics.median(kv[1])):
    us = statistics.median(ts)
    print(f"unroll {key[0]} bps {key[1]:2d} chain {key[2]}: {us:7.2f} us  {2 * n / us / 1e3:7.1f} GB/s")
