"""NEXT-2 on one GPU: cost of the fused cross-GPU combine protocol.

Times (CUDA events on the launching stream around 10 back-to-back launches,
median over batches, after warm-up):
  plain      tcr_reduce_sum_ex over the whole n (no combine)
  peer P=1   tcr_reduce_sum_peer, one-rank group (push + wait on the own mailbox)
  emulated P tcr_reduce_sum_peer_emulated: P ranks in one cooperative launch,
             each reducing n/P elements and exchanging partials through the
             mailboxes (the on-chip cost of the protocol; the NVLink latency of
             a real group is not in this number)
Sizes: 2^24 (C2, latency-bound: the protocol cost is visible), 2^30 (C3)
and 2^33 (C4's total, 16 GiB: P = 8 emulated is C4's 8-GPU problem on one GPU).
"""
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_1903_03640_b200 as tcr  # noqa: E402
import tcr_inputs as gen  # noqa: E402


def timed(fn, boxes, reps=50, warm=5):
    # a group's mailboxes must have seen the same sequence of combines:
    # restart every configuration from zeroed mailboxes
    for b in boxes:
        tcr.tcr_peer_mailbox_reset(b)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    # back-to-back launches between the events, so that host submission
    # latency (Python + ctypes) is hidden and the number is device time
    ts = []
    for _ in range(reps // 10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)  # let the host queue the batch
        a.record(s)
        for _ in range(10):
            fn()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / 10)
    return statistics.median(ts)


def main():
    boxes = [tcr.tcr_peer_mailbox_alloc() for _ in range(tcr.TCR_MAX_PEERS)]
    res = {}
    for logn in (24, 30, 33):
        n = 1 << logn
        x = gen.generate_tensor(gen.SEED_C3, 0, n, gen.UNIFORM_PM1)
        o = torch.empty(8, dtype=torch.float64, device="cuda")
        reps = 20 if logn >= 33 else 50
        r = {}
        # r02: both fused kernels (mma.sync, tcgen05) against their plain twins
        for algo in ("mma_sync", "tcgen05"):
            r[f"{algo}_plain_us"] = timed(
                lambda: tcr.tcr_reduce_sum_ex(x, out_f64=o[:1], algo=algo), boxes, reps)
            r[f"{algo}_peer_P1_us"] = timed(
                lambda: tcr.tcr_reduce_sum_peer(x, boxes[:1], 0, out_f64=o[:1], algo=algo), boxes, reps)
            for P in (1, 2, 4, 8):
                r[f"{algo}_emulated_P{P}_us"] = timed(
                    lambda: tcr.tcr_reduce_sum_peer_emulated(x, boxes[:P], out_f64=o[:P], algo=algo),
                    boxes, reps)
        r["plain_us"] = r["mma_sync_plain_us"]
        r["emulated_P8_us"] = r["mma_sync_emulated_P8_us"]
        r["gbs_plain"] = 2 * n / (r["plain_us"] * 1e-6) / 1e9
        r["gbs_emulated_P8"] = 2 * n / (r["emulated_P8_us"] * 1e-6) / 1e9
        res[f"n=2^{logn}"] = r
        del x
    torch.cuda.synchronize()
    assert not any(tcr.tcr_peer_mailbox_error(b) for b in boxes)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
