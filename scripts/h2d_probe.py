"""PCIe H2D bandwidth probe (pinned host -> device): one stream vs two / four
streams of equal parts, 2 GiB total, CUDA events, best of 5."""
import torch

n = 2 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for parts in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(parts)]
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step = n // parts
        for k, s in enumerate(streams):
            s.wait_event(a)
            with torch.cuda.stream(s):
                d[k * step:(k + 1) * step].copy_(h[k * step:(k + 1) * step], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    print(f"parts={parts}: {n / (best * 1e-3) / 1e9:.1f} GB/s")
