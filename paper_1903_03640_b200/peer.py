"""NEXT-2: the sharded reduction with the cross-GPU combine fused into the
kernel (include/tcr.h "Fused cross-GPU combine"; the paper's distributed
reduction, §II).

``PeerGroup`` owns this rank's mailbox, maps the peers' mailboxes through
CUDA IPC (handles exchanged once over the torch.distributed process group --
host plumbing, not the data path).  The epoch that tags each combine is
counted on the device, in the mailbox.  ``reduce_sum`` is ONE
launch per rank: the local reduction, the NVLink push of the fp64 partial,
the wait for the peers' partials and the rank-ordered sum -- no NCCL call,
no host synchronisation.  Every rank gets the bitwise identical total.

``lib`` and ``all_gather`` are parameters so the host logic runs under gloo
on CPU (tests/test_multigpu_gloo.py); their defaults are the library's entry
points and ``torch.distributed.all_gather_object``.
"""
from __future__ import annotations


class PeerGroup:
    def __init__(self, group=None, lib=None, all_gather=None):
        import torch.distributed as dist

        if lib is None:
            import paper_1903_03640_b200 as lib
        self._lib = lib
        self.group = group
        if dist.is_initialized():
            self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        else:
            self.rank, self.world = 0, 1
        if self.world > lib.TCR_MAX_PEERS:
            raise ValueError(f"peer group of {self.world} ranks > TCR_MAX_PEERS={lib.TCR_MAX_PEERS}")
        if all_gather is None:
            def all_gather(obj):
                out = [None] * self.world
                dist.all_gather_object(out, obj, group=group)
                return out
        # Every rank takes part in the handle exchange even if its own set-up
        # failed (it sends None), so a failure cannot leave the others blocked
        # in the collective; then all ranks raise together.
        self.mailbox, handle, err = None, None, None
        try:
            self.mailbox = lib.tcr_peer_mailbox_alloc()
            handle = lib.tcr_peer_ipc_handle(self.mailbox) if self.world > 1 else b""
        except Exception as e:
            err = e
        handles = all_gather(handle) if self.world > 1 else [handle]
        if err is not None or any(h is None for h in handles):
            if self.mailbox is not None:
                lib.tcr_peer_mailbox_free(self.mailbox)
            bad = [r for r, h in enumerate(handles) if h is None]
            raise RuntimeError(f"peer group set-up failed on rank(s) {bad}: {err!r}")
        self._opened = []
        self.mailboxes = []
        for r in range(self.world):
            if r == self.rank:
                self.mailboxes.append(self.mailbox)
            else:
                p = lib.tcr_peer_ipc_open(handles[r])
                self._opened.append(p)
                self.mailboxes.append(p)
        self.calls = 0

    def reduce_sum(self, x_local, out_f32=None, out_f64=None, algo="default", stream=None):
        """Group total of every rank's shard into out_f32 / out_f64 (device,
        1 element each), replicated on all ranks.  Every rank must call it
        the same number of times, in the same order, stream-ordered.  algo:
        "default" (by shard size: tcgen05 from 1 GiB, else mma_sync),
        "mma_sync", "tcgen05" or "shuffle"."""
        self.calls += 1
        self._lib.tcr_reduce_sum_peer(x_local, self.mailboxes, self.rank, out_f32=out_f32,
                                      out_f64=out_f64, algo=algo, stream=stream)
        return out_f32 if out_f32 is not None else out_f64

    def reduce_sum_exact(self, x_local, out_f32=None, out_f64=None, acc=None, stream=None):
        """Bitwise-exact group total (NEXT-3 limbs combined in the kernel):
        identical on every rank and for every number of ranks.  binary16 only
        (the fused exact combine kernel decodes binary16; other types raise)."""
        self._lib._require_binary16(x_local, "PeerGroup.reduce_sum_exact")
        self.calls += 1
        self._lib.tcr_reduce_sum_exact_peer(x_local, self.mailboxes, self.rank, acc=acc,
                                            out_f32=out_f32, out_f64=out_f64, stream=stream)
        return out_f32 if out_f32 is not None else out_f64

    def timed_out(self) -> bool:
        """True if a combine on this rank gave up waiting for a peer (synchronous)."""
        return self._lib.tcr_peer_mailbox_error(self.mailbox)

    def reset(self, barrier=None, stream=None) -> None:
        """Clear the error word and restart the device-side combine count
        (e.g. after a timeout).  Collective: all ranks, no combine in flight."""
        self._barrier(barrier)
        self._lib.tcr_peer_mailbox_reset(self.mailbox, stream)
        self._barrier(barrier)

    def close(self, barrier=None) -> None:
        """Quiesce, unmap the peers' mailboxes and free the own one (collective)."""
        if self.mailbox is None:
            return
        self._barrier(barrier)  # no peer still pushes into our mailbox
        for p in self._opened:
            self._lib.tcr_peer_ipc_close(p)
        self._opened = []
        self._barrier(barrier)  # no peer still maps our mailbox
        self._lib.tcr_peer_mailbox_free(self.mailbox)
        self.mailbox = None
        self.mailboxes = []

    def _barrier(self, barrier):
        import torch.distributed as dist

        if barrier is not None:
            barrier()
            return
        try:
            import torch

            if torch.cuda.is_available():
                torch.cuda.synchronize()
        except Exception:  # pragma: no cover
            pass
        if dist.is_initialized() and self.world > 1:
            dist.barrier(group=self.group)
