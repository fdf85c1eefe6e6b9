"""Small invocations of every kernel (run under compute-sanitizer --tool memcheck):
flat reductions (all algos, ragged + misaligned), segmented/batched, host entry, probes."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402

dev = "cuda"
for n in (0, 1, 7, 300, 4096 + 3, (1 << 20) + 77):
    bits = gen.generate(1, 0, n, gen.UNIFORM_PM1)
    buf = torch.empty(n + 16, dtype=torch.int16, device=dev)
    for off in (0, 3):
        x = buf[off:off + n]
        if n:
            x.copy_(torch.from_numpy(bits.view(np.int16)))
        xh = x.view(torch.float16)
        o32 = torch.empty(1, dtype=torch.float32, device=dev)
        o64 = torch.empty(1, dtype=torch.float64, device=dev)
        for algo in ("mma_sync", "tcgen05", "shuffle"):
            tcr.tcr_reduce_sum_algo(xh, out_f32=o32, out_f64=o64, algo=algo)
torch.cuda.synchronize()
# the tcgen05 dynamic tail at small sizes (forced on: its default gate is >= 32 chunks per CTA)
tcr.tcr_set_config(tcr.TCR_CFG_TC05_DYN_MIN_RUN, 0)
for dyn in (8, 100):
    tcr.tcr_set_config(tcr.TCR_CFG_TC05_DYNAMIC, dyn)
    for n in (5, 16384 * 3 + 7, (1 << 21) + 9):
        xh = torch.from_numpy(gen.generate(3, 0, n, gen.UNIFORM_PM1).view(np.int16)).to(dev).view(torch.float16)
        tcr.tcr_reduce_sum_algo(xh, out_f32=o32, out_f64=o64, algo="tcgen05")
tcr.tcr_set_config(tcr.TCR_CFG_TC05_DYNAMIC, 8)
tcr.tcr_set_config(tcr.TCR_CFG_TC05_DYN_MIN_RUN, 32)
torch.cuda.synchronize()
n = 100_000
bits = gen.generate(2, 0, n, gen.WIDE)
x = torch.from_numpy(bits.view(np.int16)).to(dev).view(torch.float16)
off = torch.tensor([0, 0, 1, 9, 300, 4097, 50_000, n], dtype=torch.int64, device=dev)
out = torch.empty(7, dtype=torch.float32, device=dev)
tcr.tcr_reduce_sum_segmented(x, off, out)
tcr.tcr_reduce_sum_segmented_shuffle(x, off, out)
outb = torch.empty(97, dtype=torch.float32, device=dev)
tcr.tcr_reduce_sum_batched(x, 1000, outb)
tcr.tcr_reduce_sum_batched_shuffle(x, 1000, outb)
print("host", tcr.tcr_reduce_sum_host(bits[:5000]))
a = torch.zeros(128 * 16, dtype=torch.int16, device=dev)
c = torch.zeros(128, dtype=torch.float32, device=dev)
d = torch.empty(128, dtype=torch.float32, device=dev)
tcr.tcr_probe_mma(a, c, d, algo="mma_sync")
tcr.tcr_probe_mma(a, c, d, algo="tcgen05")
torch.cuda.synchronize()
print("sanitize smoke done")
