"""Fresh-process warm-up study, part 2: is the slow-first-passes effect per
buffer (page level) or per process, and does it decay with passes or time?
  newbuf  -- warm x (100 launches), then a NEW 2 GiB buffer x2: 60 launches on x2
  sleepy  -- 60 launches on a fresh x, 5 ms idle + sync between launches
  write30 -- 30 generator passes over x (writes only), then 60 launches
  read1   -- one torch read pass over x (x.view(int16).sum()), then 60 launches
  read30  -- 30 torch read passes, then 60 launches"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402

variant = sys.argv[1]
torch.cuda.set_device(0)
N = 1 << 30
x = gen.generate_tensor(gen.SEED_C3, 0, N, gen.UNIFORM_PM1)
out = torch.empty(1, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
torch.cuda.synchronize()


def launches(t, k, sleep=0.0):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
    with torch.cuda.stream(s):
        for a, b in ev:
            a.record(s)
            tcr.tcr_reduce_sum_ex(t, out_f32=out, stream=s)
            b.record(s)
            if sleep:
                torch.cuda.synchronize()
                time.sleep(sleep)
    torch.cuda.synchronize()
    return [round(a.elapsed_time(b) * 1e3, 1) for a, b in ev]


target = x
if variant == "newbuf":
    launches(x, 100)
    target = gen.generate_tensor(gen.SEED_C3 + 1, 0, N, gen.UNIFORM_PM1)
elif variant == "write30":
    for _ in range(30):
        gen.generate_device(x.data_ptr(), gen.SEED_C3, 0, N, gen.UNIFORM_PM1,
                            torch.cuda.current_stream().cuda_stream)
elif variant in ("read1", "read30"):
    for _ in range(1 if variant == "read1" else 30):
        x.view(torch.int16).sum()
torch.cuda.synchronize()
launches(target, 1)  # module load
d = launches(target, 60, 0.005 if variant == "sleepy" else 0.0)
print(json.dumps({"variant": variant, "us": d, "mean_0_5": sum(d[:5]) / 5,
                  "mean_5_25": sum(d[5:25]) / 20, "mean_25_60": sum(d[25:]) / 35}))
