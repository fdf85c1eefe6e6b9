"""r02 §16: tcgen05 ring shapes with the dynamic tail, back to back (the
driver's bench shape: rounds of 20 launches between two events, median of 8
interleaved rounds) and isolated (behind a 40 us spin, median of 20).
Shapes are stages x KiB (4 accumulators, chain = KiB / 16); a ring of at most
~113 KiB lets the next launch's CTA become resident on an SM while the
current one drains (PDL overlap of its set-up).
Usage: python scripts/tc05_shape_ab.py [log2 n ...]   (default 30)"""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402

sizes = [int(a) for a in sys.argv[1:]] or [30]
K = tcr
keys = (K.TCR_CFG_TC05_STAGES, K.TCR_CFG_TC05_STAGE_KB, K.TCR_CFG_TC05_SLOTS, K.TCR_CFG_TC05_CHAIN,
        K.TCR_CFG_TC05_CTAS_PER_SM)
saved = [tcr.tcr_get_config(k) for k in keys]
arms = [("mma_sync", None)] + [(f"{st}x{kb} ct{ct}", (st, kb, 4, kb // 16, ct))
                               for st, kb, ct in ((4, 32, 1), (3, 32, 1), (3, 32, 2), (6, 16, 1),
                                                  (6, 16, 2), (4, 16, 2), (2, 64, 1), (5, 32, 1))]
out = torch.empty(1, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()


def setup(cfg):
    for k, v in zip(keys, cfg or saved):
        tcr.tcr_set_config(k, v)
    return "mma_sync" if cfg is None else "tcgen05"


def b2b(x, algo, k=20):
    with torch.cuda.stream(s):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(k):
            tcr.tcr_reduce_sum_algo(x, out_f32=out, algo=algo, stream=s)
        b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / k


def isolated(x, algo):
    with torch.cuda.stream(s):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(int(40e-6 * 1.9e9))
        a.record(s)
        tcr.tcr_reduce_sum_algo(x, out_f32=out, algo=algo, stream=s)
        b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3


for lg in sizes:
    n = 1 << lg
    x = gen.generate_tensor(gen.SEED_C3, 0, n, gen.UNIFORM_PM1)
    for name, cfg in arms:
        b2b(x, setup(cfg), 30)
    res = {name: [] for name, _ in arms}
    iso = {name: [] for name, _ in arms}
    for r in range(8):
        for name, cfg in arms:
            res[name].append(b2b(x, setup(cfg)))
    for r in range(20):
        for name, cfg in arms:
            iso[name].append(isolated(x, setup(cfg)))
    base, ibase = statistics.median(res["mma_sync"]), statistics.median(iso["mma_sync"])
    print(f"2^{lg}: back to back (20 launches, median of 8) | isolated (median of 20)")
    for name, _ in arms:
        m, mi = statistics.median(res[name]), statistics.median(iso[name])
        print(f"  {name:12s} {m:9.2f} us {2 * n / m / 1e3:6.0f} GB/s {m / base:.3f}x mma | "
              f"{mi:9.2f} us {mi / ibase:.3f}x mma", flush=True)
    del x
    torch.cuda.empty_cache()
setup(None)
