"""Library comparison point (not part of the product): torch.sum of 2^30 fp16
with fp32 accumulation, CUDA-event timed, best of 20."""
import torch
x = torch.empty(1 << 30, dtype=torch.float16, device="cuda").uniform_(-1, 1)
for _ in range(3):
    torch.sum(x, dtype=torch.float32)
ts = []
for _ in range(20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); torch.sum(x, dtype=torch.float32); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ms = min(ts)
print(f"torch.sum fp16->fp32 n=2^30: {ms*1e3:.1f} us, {2*(1<<30)/ms/1e6:.1f} GB/s, {(1<<30)/ms/1e6:.1f} Gelem/s")
