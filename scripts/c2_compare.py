"""BASELINE config 2: n = 2^24 fp16 (32 MiB, fits in the 126 MB L2) -- MMA
paths vs the warp-shuffle path.
  cold: a 512 MiB buffer is written between timed launches (outside the
        events; its dirty lines are written back during the timed kernel);
        per-launch CUDA-event time, median of 200.  Every timed launch is
        queued behind a 40 us spin kernel (torch.cuda._sleep), so the host's
        launch cost is hidden (r02; r01's numbers included it); the launch
        floor of the event pair is reported as "empty" (an empty torch op).
  cold_clean: the same with the 512 MiB buffer READ instead (L2 left full of
        clean lines: no write-back inside the timed kernel).
  warm: 100 back-to-back launches captured in a CUDA graph, replay time / 100
        (no host launch gaps; the input stays in L2).
Library calls only."""
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402

n = 1 << 24
x = gen.generate_tensor(gen.SEED_C2, 0, n, gen.UNIFORM_PM1)
out = torch.empty(1, dtype=torch.float32, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
res = {}
def graph_time(fn, reps=100):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()  # first call on this stream allocates the library workspace
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / (5 * reps)


flush16 = flush.view(torch.float16)
fout = torch.empty(1, dtype=torch.float32, device="cuda")


def cold_time(fn, clean):
    ts = []
    for i in range(230):
        if clean:
            tcr.tcr_reduce_sum_algo(flush16, out_f32=fout, algo="mma_sync")  # read-only sweep
        else:
            flush.fill_(i & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(80000)  # ~40 us at 1.9 GHz: the host enqueues fn() meanwhile
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i >= 30:
            ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


pdl_modes = [1, 0] if hasattr(tcr, "TCR_CFG_PDL") else [None]
empty = torch.empty(1, device="cuda")
res["empty:cold_clean"] = {"us": cold_time(lambda: empty.zero_(), True)}
print(f"empty op  cold_clean: {res['empty:cold_clean']['us']:7.2f} us  (event-pair launch floor)")
for pdl, algo in [(p, a) for p in pdl_modes for a in ("mma_sync", "tcgen05", "shuffle")]:
    if pdl is not None:
        tcr.tcr_set_config(tcr.TCR_CFG_PDL, pdl)
    tag = algo if pdl is None else f"{algo}/pdl{pdl}"
    fn = lambda: tcr.tcr_reduce_sum_algo(x, out_f32=out, algo=algo)  # noqa: E731
    for mode, us in (("cold", cold_time(fn, False)), ("cold_clean", cold_time(fn, True)),
                     ("warm", graph_time(lambda: tcr.tcr_reduce_sum_algo(x, out_f32=out, algo=algo)))):
        res[f"{tag}:{mode}"] = {"us": us, "GB/s": 2 * n / (us * 1e-6) / 1e9, "Gelem/s": n / (us * 1e-6) / 1e9}
        print(f"{tag:14s} {mode:10s}: {us:7.2f} us  {2*n/(us*1e-6)/1e9:8.1f} GB/s  {n/(us*1e-6)/1e9:8.1f} Gelem/s")
# torch.sum as a library reference point
tfn = lambda: torch.sum(x, dtype=torch.float32)  # noqa: E731
for mode, us in (("cold", cold_time(tfn, False)), ("cold_clean", cold_time(tfn, True)),
                 ("warm", graph_time(tfn))):
    res[f"torch.sum:{mode}"] = {"us": us, "GB/s": 2 * n / (us * 1e-6) / 1e9}
    print(f"torch.sum {mode:10s}: {us:7.2f} us  {2*n/(us*1e-6)/1e9:8.1f} GB/s")
json.dump(res, open("gpurun_out/c2_compare.json", "w"), indent=1)
