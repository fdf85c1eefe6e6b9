"""Small driver for ncu captures: runs one named kernel a few times on the
synthetic workload.  Usage: python scripts/profile_targets.py <target>
targets: c3_mma c3_tcgen05 c3_shuffle c3_exact c5 rows256 fp8_tcgen05 bf16_mma
         c2_mma c2_tcgen05 c2_shuffle (n = 2^24, BASELINE config 2)"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402

t = sys.argv[1]
out = torch.empty(1 << 20, dtype=torch.float32, device="cuda")
if t.startswith("c2_"):
    x = gen.generate_tensor(gen.SEED_C2, 0, 1 << 24, gen.UNIFORM_PM1)
    for _ in range(5):
        tcr.tcr_reduce_sum_algo(x, out_f32=out, algo={"mma": "mma_sync"}.get(t[3:], t[3:]))
elif t.startswith("c3_"):
    x = gen.generate_tensor(gen.SEED_C3, 0, 1 << 30, gen.UNIFORM_PM1)
    for _ in range(3):
        if t == "c3_exact":
            tcr.tcr_reduce_sum_exact(x, out_f32=out)
        else:
            tcr.tcr_reduce_sum_algo(x, out_f32=out, algo={"mma": "mma_sync"}.get(t[3:], t[3:]))
elif t == "c5":
    S = 1 << 20
    off = gen.offsets_from_lengths(gen.loguniform_lengths(gen.SEED_C5, S))
    x = gen.generate_tensor(gen.SEED_C5, 0, int(off[-1]), gen.UNIFORM_PM1)
    toff = torch.from_numpy(off).cuda()
    for _ in range(3):
        tcr.tcr_reduce_sum_segmented(x, toff, out)
elif t == "rows256":
    x = gen.generate_tensor(gen.SEED_C5, 0, 256 << 20, gen.UNIFORM_PM1)
    for _ in range(3):
        tcr.tcr_reduce_sum_batched(x, 256, out)
elif t == "fp8_tcgen05":
    x = gen.generate_tensor_fp8(gen.SEED_C3, 0, 1 << 31, gen.UNIFORM_PM1, gen.FP8_E4M3)
    for _ in range(3):
        tcr.tcr_reduce_sum_ex(x, out_f32=out, algo="tcgen05")
elif t == "bf16_mma":
    x = gen.generate_tensor(gen.SEED_C3, 0, 1 << 30, gen.UNIFORM_PM1, bf16=True)
    for _ in range(3):
        tcr.tcr_reduce_sum_ex(x, out_f32=out, algo="mma_sync")
torch.cuda.synchronize()
print("done", t, float(out[0].item()))
