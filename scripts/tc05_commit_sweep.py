"""tcgen05 kernel configurations that commit less often (r02: a tcgen05.commit
costs the issuing thread ~0.5 us, an MMA ~7 ns -- scripts/tc05_floor.cu).
Per config: 2^24 warm (CUDA graph of 100 launches) and 2^30 (30 back-to-back
launches between one event pair), mma.sync as the reference on the same box.
Config = (stages, stage KiB, slots, chain, CTAs/SM)."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402
from c2_compare_lib import graph_time  # noqa: E402

x24 = gen.generate_tensor(gen.SEED_C2, 0, 1 << 24, gen.UNIFORM_PM1)
x30 = gen.generate_tensor(gen.SEED_C3, 0, 1 << 30, gen.UNIFORM_PM1)
out = torch.empty(1, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()


def b2b(x, algo, k=30):
    with torch.cuda.stream(s):
        for _ in range(3):
            tcr.tcr_reduce_sum_algo(x, out_f32=out, algo=algo, stream=s)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(k):
            tcr.tcr_reduce_sum_algo(x, out_f32=out, algo=algo, stream=s)
        b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / k


keys = (tcr.TCR_CFG_TC05_STAGES, tcr.TCR_CFG_TC05_STAGE_KB, tcr.TCR_CFG_TC05_SLOTS,
        tcr.TCR_CFG_TC05_CHAIN, tcr.TCR_CFG_TC05_CTAS_PER_SM)
default = tuple(tcr.tcr_get_config(k) for k in keys)
m24 = statistics.median(graph_time(lambda: tcr.tcr_reduce_sum_algo(x24, out_f32=out, algo="mma_sync"))
                        for _ in range(3))
m30 = b2b(x30, "mma_sync")
print(f"mma_sync reference: 2^24 warm {m24:.2f} us, 2^30 {m30:.1f} us ({2 ** 31 / m30 / 1e3:.0f} GB/s)",
      flush=True)
configs = [default, (3, 64, 4, 4, 1), (2, 64, 4, 4, 1), (4, 32, 4, 2, 1), (6, 32, 4, 2, 1), (4, 16, 4, 1, 3),
           (2, 32, 4, 2, 3), (3, 32, 4, 2, 2), (8, 16, 4, 1, 1), (3, 64, 4, 4, 2),
           (3, 48, 4, 4, 1)]
for cfg in configs:
    for k, v in zip(keys, cfg):
        tcr.tcr_set_config(k, v)
    t24 = statistics.median(graph_time(lambda: tcr.tcr_reduce_sum_algo(x24, out_f32=out, algo="tcgen05"))
                            for _ in range(3))
    t30 = b2b(x30, "tcgen05")
    print(f"tcgen05 stages={cfg[0]} kb={cfg[1]:2d} slots={cfg[2]:2d} chain={cfg[3]} ctas={cfg[4]}: "
          f"2^24 warm {t24:6.2f} us ({t24 / m24:.2f}x mma)  2^30 {t30:6.1f} us "
          f"({2 ** 31 / t30 / 1e3:.0f} GB/s, {t30 / m30:.3f}x mma)", flush=True)
for k, v in zip(keys, default):
    tcr.tcr_set_config(k, v)
