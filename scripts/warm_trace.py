"""Per-launch durations of the default C3 kernel from a cold start (after an
idle pause), to explain the 20-step vs 1000-step gap.
Each launch bracketed by its own CUDA event pair (adds a small gap; only the
trend matters).  Also samples NVML SM / memory clocks and power."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402

import pynvml  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
torch.cuda.set_device(0)
x = gen.generate_tensor(gen.SEED_C3, 0, 1 << 30, gen.UNIFORM_PM1)
out = torch.empty(1, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
res = {}
for label, pre in (("idle2s", None), ("idle2s_again", None), ("after_50ms_busy", 50), ("after_300ms_busy", 300)):
    torch.cuda.synchronize()
    time.sleep(2.0)
    if pre:
        a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
        t0 = time.time()
        while time.time() - t0 < pre / 1e3:
            a @ a
        torch.cuda.synchronize()
    clk0 = (pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM))
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(400)]
    with torch.cuda.stream(s):
        for a_, b_ in ev:
            a_.record(s)
            tcr.tcr_reduce_sum_ex(x, out_f32=out, stream=s)
            b_.record(s)
    torch.cuda.synchronize()
    d = [a_.elapsed_time(b_) * 1e3 for a_, b_ in ev]
    clk1 = (pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM))
    res[label] = {"us": [round(v, 1) for v in d], "clk_before": clk0, "clk_after": clk1}
    print(label, clk0, clk1, "first 30:", [round(v, 1) for v in d[:30]])
    print("  mean 0-5", sum(d[:5]) / 5, "5-25", sum(d[5:25]) / 20, "25-100", sum(d[25:100]) / 75,
          "100-400", sum(d[100:]) / 300)
json.dump(res, open("gpurun_out/warm_trace.json", "w"))
