"""r02 §18: the exact reduction fused with the peer limb combine, one real rank
(nranks = 1) at 2^30 and 8 emulated ranks over 2^33: the LDG peer kernel
(TCR_CFG_EXACT_BULK = 0) vs the TMA-fed one, back to back (10 launches,
median of 5 interleaved rounds)."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402

# one mailbox set per group: a mailbox's epoch counts the combines of ITS group
boxes1 = [tcr.tcr_peer_mailbox_alloc()]
boxes8 = [tcr.tcr_peer_mailbox_alloc() for _ in range(8)]
s = torch.cuda.Stream()


def b2b(f, k=10):
    with torch.cuda.stream(s):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(k):
            f()
        b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / k


for lg, P in ((30, 1), (33, 8)):
    n = 1 << lg
    x = gen.generate_tensor(gen.SEED_C4, 0, n, gen.UNIFORM_PM1)
    o32 = torch.empty(P, dtype=torch.float32, device="cuda")
    if P == 1:
        f = lambda: tcr.tcr_reduce_sum_exact_peer(x, boxes1, 0, out_f32=o32, stream=s)  # noqa: E731
    else:
        f = lambda: tcr.tcr_reduce_sum_exact_peer_emulated(x, boxes8, out_f32=o32, stream=s)  # noqa: E731
    res = {}
    for r in range(5):
        for name, eb in (("ldg", 0), ("bulk", 1)):
            tcr.tcr_set_config(tcr.TCR_CFG_EXACT_BULK, eb)
            if r == 0:
                b2b(f, 3)
            res.setdefault(name, []).append(b2b(f))
    tcr.tcr_set_config(tcr.TCR_CFG_EXACT_BULK, 1)
    print(f"exact peer 2^{lg} P={P}: " + " | ".join(
        f"{k} {statistics.median(v):9.2f} us {2 * n / statistics.median(v) / 1e3:6.0f} GB/s" for k, v in res.items()),
        flush=True)
    del x
    torch.cuda.empty_cache()
