"""Fresh-process warm-up study: per-launch durations of
the default C3 kernel for the first 60 launches of a NEW process, after one
of several pre-phases.  Usage: python scripts/warm_fresh.py <variant>
  none   -- nothing between input generation and the launches
  spin   -- 30 ms of a compute-only kernel (torch.cuda._sleep)
  copy   -- 30 ms of device-to-device copies (HBM traffic, another kernel)
  e2e    -- one host-entry call (tcr_reduce_sum_host_ex over the same bits)
  self   -- 100 launches of the kernel itself first (a long warm-up)"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402

variant = sys.argv[1]
algo = sys.argv[2] if len(sys.argv) > 2 else "default"
torch.cuda.set_device(0)
x = gen.generate_tensor(gen.SEED_C3, 0, 1 << 30, gen.UNIFORM_PM1)
out = torch.empty(1, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
if variant == "spin":
    torch.cuda._sleep(int(30e-3 * 1.9e9))
elif variant == "copy":
    y = torch.empty_like(x)
    while time.perf_counter() - t0 < 0.03:
        y.copy_(x)
        torch.cuda.synchronize()
elif variant == "e2e":
    host = torch.empty(2 << 30, dtype=torch.uint8, pin_memory=True)
    host.copy_(x.view(torch.uint8))
    tcr.tcr_reduce_sum_host_ex(host, tcr.TCR_DTYPE_F16, n=1 << 30)
elif variant == "self":
    with torch.cuda.stream(s):
        for _ in range(100):
            tcr.tcr_reduce_sum_ex(x, out_f32=out, algo=algo, stream=s)
torch.cuda.synchronize()
pre_ms = (time.perf_counter() - t0) * 1e3
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(60)]
with torch.cuda.stream(s):
    for a, b in ev:
        a.record(s)
        tcr.tcr_reduce_sum_ex(x, out_f32=out, algo=algo, stream=s)
        b.record(s)
torch.cuda.synchronize()
d = [round(a.elapsed_time(b) * 1e3, 1) for a, b in ev]
print(json.dumps({"variant": variant, "algo": algo, "pre_ms": round(pre_ms, 1), "us": d,
                  "mean_1_6": sum(d[1:6]) / 5, "mean_6_26": sum(d[6:26]) / 20,
                  "mean_26_60": sum(d[26:]) / 34}))
