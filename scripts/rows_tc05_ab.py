"""r02 §17: batched fixed-length rows, tcgen05 (128 segments per MMA, TMA
tensor copies) vs the mma.sync kernels, 1 GiB of binary16 per L (S = 2^29 / L),
back to back: 3 warm-up then 30 launches between one event pair, median of 5
interleaved rounds; GB/s = (2 S L + 4 S) / t."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402

Ls = [int(a) for a in sys.argv[1:]] or [8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 16384]
s = torch.cuda.Stream()
DYNS = [int(v) for v in __import__("os").environ.get("DYNS", "0 8").split()]
if __import__("os").environ.get("STAGES"):
    tcr.tcr_set_config(tcr.TCR_CFG_ROWS_TC05_STAGES, int(__import__("os").environ["STAGES"]))
print("rows_tc05 stages", tcr.tcr_get_config(tcr.TCR_CFG_ROWS_TC05_STAGES), flush=True)


def run(x, L, out, k=30):
    with torch.cuda.stream(s):
        for _ in range(3):
            tcr.tcr_reduce_sum_batched_ex(x, L, out, algo="mma_sync", stream=s)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(k):
            tcr.tcr_reduce_sum_batched_ex(x, L, out, algo="mma_sync", stream=s)
        b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / k


dt = __import__("os").environ.get("DTYPE", "f16")
es = 1 if dt in ("e4m3", "e5m2") else 2
for L in Ls:
    S = (1 << 30) // es // L
    if es == 1:
        x = gen.generate_tensor_fp8(gen.SEED_C5, 0, L * S, gen.UNIFORM_PM1,
                                    gen.FP8_E4M3 if dt == "e4m3" else gen.FP8_E5M2)
    else:
        x = gen.generate_tensor(gen.SEED_C5, 0, L * S, gen.UNIFORM_PM1, bf16=(dt == "bf16"))
    out = torch.empty(S, dtype=torch.float32, device="cuda")
    arms = [(0, 8)] + [(1, d) for d in DYNS]  # (rows_tc05, dynamic %)
    res = {a: [] for a in arms}
    for r in range(5):
        for on, d in arms:
            tcr.tcr_set_config(tcr.TCR_CFG_ROWS_TC05, on)
            tcr.tcr_set_config(tcr.TCR_CFG_TC05_DYNAMIC, d)
            res[(on, d)].append(run(x, L, out))
    tcr.tcr_set_config(tcr.TCR_CFG_ROWS_TC05, 1)
    tcr.tcr_set_config(tcr.TCR_CFG_TC05_DYNAMIC, 8)
    gb = lambda us: (es * S * L + 4 * S) / (us * 1e-6) / 1e9  # noqa: E731
    m0 = statistics.median(res[(0, 8)])
    line = f"L={L:6d} S={S:9d}  mma.sync {m0:8.1f} us {gb(m0):7.1f} GB/s"
    for on, d in arms[1:]:
        m = statistics.median(res[(on, d)])
        line += f" | tc05 dyn{d} {m:8.1f} us {gb(m):7.1f} GB/s {m / m0:.3f}"
    print(line, flush=True)
    del x, out
    torch.cuda.empty_cache()
