"""paper_1903_03640_b200 -- B200-native tensor-core (MMA-encoded) fp16 sum
reduction, from scratch, after arXiv 1903.03640 ("Analyzing GPU Tensor Core
Potential for Fast Reductions").

This module is the thin Python binding of ``libtcr.so`` (C ABI declared in
``include/tcr.h``): argument marshalling only.  Every step of the reduction
runs in the library's sm_100a kernels; there is no CPU or library fallback,
and importing this module fails loudly if ``libtcr.so`` is missing.

Functions take either torch CUDA tensors (dtype float16 / int64 / float32 /
float64) or raw device pointers (ints), and a CUDA stream (torch.cuda.Stream,
a raw handle int, or None for torch's current stream).

Names follow the C ABI:

* :func:`tcr_reduce_sum`, :func:`tcr_reduce_sum_shuffle`,
  :func:`tcr_reduce_sum_f64`, :func:`tcr_reduce_sum_algo`
* :func:`tcr_reduce_sum_segmented`, :func:`tcr_reduce_sum_segmented_shuffle`
* :func:`tcr_reduce_sum_batched`, :func:`tcr_reduce_sum_batched_shuffle`
* :func:`tcr_reduce_sum_host` (host buffers, end to end)
* :func:`tcr_round_f64_to_f32`, :func:`tcr_probe_mma`
* :func:`tcr_set_config` / :func:`tcr_get_config`, :func:`tcr_launch_count`,
  :func:`tcr_release_workspaces`, :func:`tcr_version`
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtcr.so")

TCR_OK = 0
TCR_ERR_INVALID_VALUE = 1
TCR_ERR_UNSUPPORTED_DEVICE = 2
TCR_ERR_OUT_OF_MEMORY = 3
TCR_ERR_CUDA = 4

TCR_ALGO_DEFAULT = 0
TCR_ALGO_MMA_SYNC = 1
TCR_ALGO_TCGEN05 = 2
TCR_ALGO_SHUFFLE = 3
TCR_ALGO_BULK_MMA = 4
ALGOS = {"default": 0, "mma_sync": 1, "tcgen05": 2, "shuffle": 3, "bulk": 4}
TCR_DTYPE_F16 = 0
TCR_DTYPE_BF16 = 1
TCR_DTYPE_E4M3 = 2
TCR_DTYPE_E5M2 = 3

TCR_CFG_DEFAULT_ALGO = 0
TCR_CFG_BLOCKS_PER_SM = 1
TCR_CFG_UNROLL = 2
TCR_CFG_TC05_STAGES = 3
TCR_CFG_TC05_STAGE_KB = 4
TCR_CFG_CHAIN = 5
TCR_CFG_TC05_SLOTS = 6
TCR_CFG_TC05_CHAIN = 7
TCR_CFG_TC05_CTAS_PER_SM = 8
TCR_CFG_TC05_PREFETCH = 9
TCR_CFG_TC05_SPLIT = 10
TCR_CFG_TC05_INTERLEAVE = 11
TCR_CFG_EXACT_UNROLL = 12
TCR_CFG_EXACT_BLOCKS_PER_SM = 13
TCR_CFG_BULK_STAGES = 14
TCR_CFG_BULK_STAGE_KB = 15
TCR_CFG_BULK_CTAS_PER_SM = 16
TCR_CFG_PEER_TIMEOUT_MS = 17
TCR_CFG_PDL = 18
TCR_CFG_TC05_DYNAMIC = 19
TCR_CFG_TC05_DYN_MIN_RUN = 20
TCR_CFG_ROWS_TC05 = 21
TCR_CFG_ROWS_TC05_STAGES = 22
TCR_CFG_EXACT_BULK = 23

TCR_EXACT_ACC_WORDS = 6
TCR_EXACT_BF16_ACC_WORDS = 27
TCR_MAX_PEERS = 8
TCR_PEER_MAILBOX_BYTES = 2048
TCR_IPC_HANDLE_BYTES = 64


class TcrError(RuntimeError):
    def __init__(self, status: int, fn: str, detail: str):
        self.status = status
        super().__init__(f"{fn} failed: {_status_name(status)}: {detail}")


if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libtcr.so not found at {LIB_PATH}; build it with "
        "`python -c 'import __graft_entry__ as g; g.build()'` (there is no fallback path)")

_lib = ctypes.CDLL(LIB_PATH)

_P = ctypes.c_void_p
_SZ = ctypes.c_size_t
_I = ctypes.c_int

_SIGS = {
    "tcr_reduce_sum": [_P, _SZ, _P, _P],
    "tcr_reduce_sum_shuffle": [_P, _SZ, _P, _P],
    "tcr_reduce_sum_f64": [_P, _SZ, _P, _P],
    "tcr_reduce_sum_algo": [_P, _SZ, _P, _P, _I, _P],
    "tcr_reduce_sum_segmented": [_P, _P, _SZ, _P, _P],
    "tcr_reduce_sum_ex": [_P, _SZ, _I, _P, _P, _I, _P],
    "tcr_reduce_sum_segmented_ex": [_P, _I, _P, _SZ, _P, _I, _P],
    "tcr_reduce_sum_batched_ex": [_P, _I, _SZ, _SZ, _P, _I, _P],
    "tcr_reduce_sum_segmented_shuffle": [_P, _P, _SZ, _P, _P],
    "tcr_reduce_sum_batched": [_P, _SZ, _SZ, _P, _P],
    "tcr_reduce_sum_batched_shuffle": [_P, _SZ, _SZ, _P, _P],
    "tcr_reduce_sum_host": [_P, _SZ, _P, _P],
    "tcr_reduce_sum_host_ex": [_P, _SZ, _I, _P, _P],
    "tcr_round_f64_to_f32": [_P, _P, _P],
    "tcr_reduce_sum_exact": [_P, _SZ, _P, _P, _P, _P],
    "tcr_exact_finalize": [_P, _P, _P, _P],
    "tcr_exact_finalize_ex": [_P, _I, _P, _P, _P],
    "tcr_reduce_sum_exact_ex": [_P, _SZ, _I, _P, _P, _P, _P],
    "tcr_probe_mma": [_P, _P, _P, _I, _P],
    "tcr_probe_collapse": [_P, _P, _I, _P],
    "tcr_reduce_sum_paper_f16": [_P, _SZ, _P, _P],
    "tcr_reduce_sum_study_fp32": [_P, _SZ, _I, _P, _P],
    "tcr_set_config": [_I, _I],
    "tcr_release_workspaces": [],
    "tcr_reduce_sum_peer": [_P, _SZ, _I, _I, _P, _I, _I, _P, _P, _P],
    "tcr_reduce_sum_peer_emulated": [_P, _SZ, _I, _I, _P, _I, _P, _P, _P],
    "tcr_reduce_sum_exact_peer": [_P, _SZ, _P, _I, _I, _P, _P, _P, _P],
    "tcr_reduce_sum_exact_peer_emulated": [_P, _SZ, _P, _I, _P, _P, _P, _P],
    "tcr_peer_mailbox_alloc": [_P],
    "tcr_peer_mailbox_free": [_P],
    "tcr_peer_mailbox_reset": [_P, _P],
    "tcr_peer_mailbox_error": [_P, _P],
    "tcr_peer_ipc_handle": [_P, _P],
    "tcr_peer_ipc_open": [_P, _P],
    "tcr_peer_ipc_close": [_P],
}
for _name, _args in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = ctypes.c_int
_lib.tcr_get_config.argtypes = [_I]
_lib.tcr_get_config.restype = ctypes.c_int
_lib.tcr_status_string.argtypes = [_I]
_lib.tcr_status_string.restype = ctypes.c_char_p
_lib.tcr_last_error.argtypes = []
_lib.tcr_last_error.restype = ctypes.c_char_p
_lib.tcr_launch_count.argtypes = []
_lib.tcr_launch_count.restype = ctypes.c_uint64
_lib.tcr_default_algo.argtypes = [_SZ, _I]
_lib.tcr_default_algo.restype = ctypes.c_int
_lib.tcr_version.argtypes = []
_lib.tcr_version.restype = ctypes.c_int


def _status_name(s: int) -> str:
    return _lib.tcr_status_string(int(s)).decode()


def _check(status: int, fn: str) -> None:
    if status != TCR_OK:
        raise TcrError(status, fn, _lib.tcr_last_error().decode())


def _ptr(t) -> int | None:
    """Device (or host) address of a tensor / int / None."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _numel(t, n):
    if n is not None:
        return int(n)
    return int(t.numel())


def _stream(stream, like=None) -> int | None:
    if stream is None:
        import torch

        dev = like.device if like is not None and hasattr(like, "device") else None
        return torch.cuda.current_stream(dev).cuda_stream or None
    if isinstance(stream, int):
        return stream or None
    return stream.cuda_stream or None


def tcr_reduce_sum(x, out, n=None, stream=None) -> None:
    """out[0] (float32, device) = sum of the n binary16 values of x (MMA-encoded)."""
    _check(_lib.tcr_reduce_sum(_ptr(x), _numel(x, n), _ptr(out), _stream(stream, x)),
           "tcr_reduce_sum")


def tcr_reduce_sum_shuffle(x, out, n=None, stream=None) -> None:
    """Classic warp-shuffle tree reduction; same contract as tcr_reduce_sum."""
    _check(_lib.tcr_reduce_sum_shuffle(_ptr(x), _numel(x, n), _ptr(out), _stream(stream, x)),
           "tcr_reduce_sum_shuffle")


def tcr_reduce_sum_f64(x, out, n=None, stream=None) -> None:
    """out[0] (float64, device) = the binary64 total before the final rounding."""
    _check(_lib.tcr_reduce_sum_f64(_ptr(x), _numel(x, n), _ptr(out), _stream(stream, x)),
           "tcr_reduce_sum_f64")


def tcr_reduce_sum_algo(x, out_f32=None, out_f64=None, algo=TCR_ALGO_DEFAULT, n=None,
                        stream=None) -> None:
    if isinstance(algo, str):
        algo = ALGOS[algo]
    _check(_lib.tcr_reduce_sum_algo(_ptr(x), _numel(x, n), _ptr(out_f32), _ptr(out_f64),
                                    int(algo), _stream(stream, x)), "tcr_reduce_sum_algo")


def _dtype_of(x, dtype):
    if dtype is not None:
        return int(dtype)
    try:
        import torch

        dt = getattr(x, "dtype", None)
        if dt == torch.bfloat16:
            return TCR_DTYPE_BF16
        if dt == torch.float8_e4m3fn:
            return TCR_DTYPE_E4M3
        if dt == torch.float8_e5m2:
            return TCR_DTYPE_E5M2
    except ImportError:  # pragma: no cover
        pass
    return TCR_DTYPE_F16


def _check_acc(acc, code: int, fn: str, ranks: int = 1) -> None:
    """An exact state must be an int64 device tensor of at least the type's
    word count (the C ABI takes a bare pointer and cannot check its length)."""
    if acc is None or isinstance(acc, int):
        return
    import torch

    words = (TCR_EXACT_BF16_ACC_WORDS if code == TCR_DTYPE_BF16 else TCR_EXACT_ACC_WORDS) * ranks
    if acc.dtype != torch.int64 or not acc.is_cuda or acc.numel() < words or not acc.is_contiguous():
        raise ValueError(f"{fn}: acc must be a contiguous int64 CUDA tensor of >= {words} words "
                         f"for this dtype (got {acc.dtype}, {acc.numel()} words, {acc.device})")


def _require_binary16(x, fn: str) -> None:
    """Entry points that take binary16 only (the fused exact peer combine)."""
    import torch

    dt = getattr(x, "dtype", None)
    if dt is not None and dt not in (torch.float16, torch.int16):
        raise ValueError(f"{fn} takes binary16 input (torch.float16), got {dt}")


def tcr_reduce_sum_ex(x, out_f32=None, out_f64=None, algo=TCR_ALGO_DEFAULT, dtype=None, n=None,
                      stream=None) -> None:
    """Sum of binary16 or bfloat16 x (dtype from the tensor unless given)."""
    if isinstance(algo, str):
        algo = ALGOS[algo]
    _check(_lib.tcr_reduce_sum_ex(_ptr(x), _numel(x, n), _dtype_of(x, dtype), _ptr(out_f32),
                                  _ptr(out_f64), int(algo), _stream(stream, x)),
           "tcr_reduce_sum_ex")


def tcr_reduce_sum_segmented_ex(x, offsets, out, algo=TCR_ALGO_DEFAULT, dtype=None,
                                num_segments=None, stream=None) -> None:
    if isinstance(algo, str):
        algo = ALGOS[algo]
    s = int(num_segments) if num_segments is not None else int(out.numel())
    _check(_lib.tcr_reduce_sum_segmented_ex(_ptr(x), _dtype_of(x, dtype), _ptr(offsets), s,
                                            _ptr(out), int(algo), _stream(stream, x)),
           "tcr_reduce_sum_segmented_ex")


def tcr_reduce_sum_batched_ex(x, segment_len, out, algo=TCR_ALGO_DEFAULT, dtype=None,
                              num_segments=None, stream=None) -> None:
    """Batched sums for any input type (segment_len in elements)."""
    if isinstance(algo, str):
        algo = ALGOS[algo]
    s = int(num_segments) if num_segments is not None else int(out.numel())
    _check(_lib.tcr_reduce_sum_batched_ex(_ptr(x), _dtype_of(x, dtype), s, int(segment_len),
                                          _ptr(out), int(algo), _stream(stream, x)),
           "tcr_reduce_sum_batched_ex")


def tcr_reduce_sum_segmented(x, offsets, out, num_segments=None, stream=None) -> None:
    """out[j] = sum of x[offsets[j]:offsets[j+1]] (CSR, int64 offsets on the device)."""
    s = int(num_segments) if num_segments is not None else int(out.numel())
    _check(_lib.tcr_reduce_sum_segmented(_ptr(x), _ptr(offsets), s, _ptr(out), _stream(stream, x)),
           "tcr_reduce_sum_segmented")


def tcr_reduce_sum_segmented_shuffle(x, offsets, out, num_segments=None, stream=None) -> None:
    s = int(num_segments) if num_segments is not None else int(out.numel())
    _check(_lib.tcr_reduce_sum_segmented_shuffle(_ptr(x), _ptr(offsets), s, _ptr(out),
                                                 _stream(stream, x)),
           "tcr_reduce_sum_segmented_shuffle")


def tcr_reduce_sum_batched(x, segment_len, out, num_segments=None, stream=None) -> None:
    """out[j] = sum of x[j*L:(j+1)*L]."""
    s = int(num_segments) if num_segments is not None else int(out.numel())
    _check(_lib.tcr_reduce_sum_batched(_ptr(x), s, int(segment_len), _ptr(out),
                                       _stream(stream, x)), "tcr_reduce_sum_batched")


def tcr_reduce_sum_batched_shuffle(x, segment_len, out, num_segments=None, stream=None) -> None:
    s = int(num_segments) if num_segments is not None else int(out.numel())
    _check(_lib.tcr_reduce_sum_batched_shuffle(_ptr(x), s, int(segment_len), _ptr(out),
                                               _stream(stream, x)),
           "tcr_reduce_sum_batched_shuffle")


def tcr_reduce_sum_host(x, n=None, stream=None) -> float:
    """End to end: x is a HOST buffer (pinned CPU tensor, numpy array or address).
    Returns the binary32 sum as a Python float (the call synchronises `stream`)."""
    res = ctypes.c_float(0.0)
    if hasattr(x, "ctypes"):  # numpy
        addr, cnt = x.ctypes.data, x.size
    else:
        addr, cnt = _ptr(x), (x.numel() if hasattr(x, "numel") else None)
    cnt = int(n) if n is not None else int(cnt)
    if stream is None:
        import torch

        stream = torch.cuda.current_stream().cuda_stream
    _check(_lib.tcr_reduce_sum_host(addr, cnt, ctypes.addressof(res), _stream(stream)),
           "tcr_reduce_sum_host")
    return float(res.value)


def tcr_reduce_sum_host_ex(x, dtype, n=None, stream=None) -> float:
    """tcr_reduce_sum_host for any input type (dtype: TCR_DTYPE_*), x a HOST
    buffer of raw element bits (pinned CPU tensor, numpy array or address)."""
    res = ctypes.c_float(0.0)
    if hasattr(x, "ctypes"):  # numpy
        addr, cnt = x.ctypes.data, x.size
    else:
        addr, cnt = _ptr(x), (x.numel() if hasattr(x, "numel") else None)
    cnt = int(n) if n is not None else int(cnt)
    if stream is None:
        import torch

        stream = torch.cuda.current_stream().cuda_stream
    _check(_lib.tcr_reduce_sum_host_ex(addr, cnt, int(dtype), ctypes.addressof(res),
                                       _stream(stream)),
           "tcr_reduce_sum_host_ex")
    return res.value


def tcr_reduce_sum_exact(x, acc=None, out_f32=None, out_f64=None, n=None, stream=None) -> None:
    """Exact sum of binary16 x: acc (int64[6] device: limbs l0,l1,l2 of the sum
    in units of 2^-24, base 2^40, then NaN/+inf/-inf counts) and/or the
    correctly rounded float32 / float64."""
    _require_binary16(x, "tcr_reduce_sum_exact")
    _check_acc(acc, TCR_DTYPE_F16, "tcr_reduce_sum_exact")
    _check(_lib.tcr_reduce_sum_exact(_ptr(x), _numel(x, n), _ptr(acc), _ptr(out_f32),
                                     _ptr(out_f64), _stream(stream, x)), "tcr_reduce_sum_exact")


def tcr_reduce_sum_exact_ex(x, acc=None, out_f32=None, out_f64=None, dtype=None, n=None,
                            stream=None) -> None:
    """Bitwise-exact sum of binary16, bfloat16 or fp8 (E4M3 / E5M2) x.  acc, if
    given, receives the mergeable exact state: TCR_EXACT_ACC_WORDS (6) int64
    for binary16 / fp8, TCR_EXACT_BF16_ACC_WORDS (27) for bfloat16 (tcr.h)."""
    code = _dtype_of(x, dtype)
    _check_acc(acc, code, "tcr_reduce_sum_exact_ex")
    _check(_lib.tcr_reduce_sum_exact_ex(_ptr(x), _numel(x, n), code, _ptr(acc),
                                        _ptr(out_f32), _ptr(out_f64), _stream(stream, x)),
           "tcr_reduce_sum_exact_ex")


def tcr_exact_finalize(acc, out_f32=None, out_f64=None, stream=None) -> None:
    """RNE float32 / float64 of an (allreduced) binary16 exact state acc[6]."""
    _check_acc(acc, TCR_DTYPE_F16, "tcr_exact_finalize")
    _check(_lib.tcr_exact_finalize(_ptr(acc), _ptr(out_f32), _ptr(out_f64), _stream(stream, acc)),
           "tcr_exact_finalize")


def tcr_exact_finalize_ex(acc, dtype, out_f32=None, out_f64=None, stream=None) -> None:
    """RNE of an (allreduced) exact state of any exact-capable dtype (6 int64
    words for binary16 / fp8, 27 for bfloat16)."""
    _check_acc(acc, int(dtype), "tcr_exact_finalize_ex")
    _check(_lib.tcr_exact_finalize_ex(_ptr(acc), int(dtype), _ptr(out_f32), _ptr(out_f64),
                                      _stream(stream, acc)),
           "tcr_exact_finalize_ex")


def tcr_round_f64_to_f32(inp, out, stream=None) -> None:
    _check(_lib.tcr_round_f64_to_f32(_ptr(inp), _ptr(out), _stream(stream, inp)),
           "tcr_round_f64_to_f32")


def tcr_probe_mma(a, c, d, algo=TCR_ALGO_MMA_SYNC, stream=None) -> None:
    if isinstance(algo, str):
        algo = ALGOS[algo]
    _check(_lib.tcr_probe_mma(_ptr(a), _ptr(c), _ptr(d), int(algo), _stream(stream, a)),
           "tcr_probe_mma")


# Fused cross-GPU combine (NEXT-2) ------------------------------------------------


def _mailbox_array(mailboxes):
    arr = (ctypes.c_void_p * len(mailboxes))(*[int(m) for m in mailboxes])
    return arr


def tcr_peer_mailbox_alloc() -> int:
    """A zeroed TCR_PEER_MAILBOX_BYTES mailbox on the current device (address)."""
    p = ctypes.c_void_p()
    _check(_lib.tcr_peer_mailbox_alloc(ctypes.byref(p)), "tcr_peer_mailbox_alloc")
    return int(p.value)


def tcr_peer_mailbox_free(mailbox: int) -> None:
    _check(_lib.tcr_peer_mailbox_free(mailbox), "tcr_peer_mailbox_free")


def tcr_peer_mailbox_reset(mailbox: int, stream=None) -> None:
    _check(_lib.tcr_peer_mailbox_reset(mailbox, _stream(stream)), "tcr_peer_mailbox_reset")


def tcr_peer_mailbox_error(mailbox: int) -> bool:
    """True if a combine on this mailbox's rank timed out (synchronous)."""
    v = ctypes.c_int()
    _check(_lib.tcr_peer_mailbox_error(mailbox, ctypes.byref(v)), "tcr_peer_mailbox_error")
    return bool(v.value)


def tcr_peer_ipc_handle(mailbox: int) -> bytes:
    buf = ctypes.create_string_buffer(TCR_IPC_HANDLE_BYTES)
    _check(_lib.tcr_peer_ipc_handle(mailbox, buf), "tcr_peer_ipc_handle")
    return buf.raw


def tcr_peer_ipc_open(handle: bytes) -> int:
    if len(handle) != TCR_IPC_HANDLE_BYTES:
        raise ValueError("IPC handle must be TCR_IPC_HANDLE_BYTES long")
    p = ctypes.c_void_p()
    _check(_lib.tcr_peer_ipc_open(ctypes.create_string_buffer(handle, len(handle)),
                                  ctypes.byref(p)), "tcr_peer_ipc_open")
    return int(p.value)


def tcr_peer_ipc_close(peer_mailbox: int) -> None:
    _check(_lib.tcr_peer_ipc_close(peer_mailbox), "tcr_peer_ipc_close")


def tcr_reduce_sum_peer(x, mailboxes, rank, out_f32=None, out_f64=None, algo=TCR_ALGO_DEFAULT,
                        dtype=None, n=None, stream=None) -> None:
    """This rank's shard reduced and combined with its peers' in one launch."""
    if isinstance(algo, str):
        algo = ALGOS[algo]
    _check(_lib.tcr_reduce_sum_peer(_ptr(x), _numel(x, n), _dtype_of(x, dtype), int(algo),
                                    _mailbox_array(mailboxes), len(mailboxes), int(rank),
                                    _ptr(out_f32), _ptr(out_f64), _stream(stream, x)),
           "tcr_reduce_sum_peer")


def tcr_reduce_sum_peer_emulated(x, mailboxes, out_f32=None, out_f64=None,
                                 algo=TCR_ALGO_DEFAULT, dtype=None, n=None, stream=None) -> None:
    """All len(mailboxes) ranks emulated in one cooperative launch (out_*[r] per rank)."""
    if isinstance(algo, str):
        algo = ALGOS[algo]
    _check(_lib.tcr_reduce_sum_peer_emulated(_ptr(x), _numel(x, n), _dtype_of(x, dtype),
                                             int(algo), _mailbox_array(mailboxes),
                                             len(mailboxes), _ptr(out_f32),
                                             _ptr(out_f64), _stream(stream, x)),
           "tcr_reduce_sum_peer_emulated")


def tcr_reduce_sum_exact_peer(x, mailboxes, rank, acc=None, out_f32=None, out_f64=None, n=None,
                              stream=None) -> None:
    """Exact sum of this rank's binary16 shard fused with the group's limb
    combine (binary16 only: other types raise)."""
    _require_binary16(x, "tcr_reduce_sum_exact_peer")
    _check_acc(acc, TCR_DTYPE_F16, "tcr_reduce_sum_exact_peer")
    _check(_lib.tcr_reduce_sum_exact_peer(_ptr(x), _numel(x, n), _mailbox_array(mailboxes),
                                          len(mailboxes), int(rank), _ptr(acc), _ptr(out_f32),
                                          _ptr(out_f64), _stream(stream, x)),
           "tcr_reduce_sum_exact_peer")


def tcr_reduce_sum_exact_peer_emulated(x, mailboxes, acc=None, out_f32=None, out_f64=None, n=None,
                                       stream=None) -> None:
    """All len(mailboxes) ranks of the exact fused combine in one cooperative
    launch (binary16 only; acc, if given, holds 6 int64 words per rank)."""
    _require_binary16(x, "tcr_reduce_sum_exact_peer_emulated")
    _check_acc(acc, TCR_DTYPE_F16, "tcr_reduce_sum_exact_peer_emulated", ranks=len(mailboxes))
    _check(_lib.tcr_reduce_sum_exact_peer_emulated(_ptr(x), _numel(x, n),
                                                   _mailbox_array(mailboxes), len(mailboxes),
                                                   _ptr(acc), _ptr(out_f32), _ptr(out_f64),
                                                   _stream(stream, x)),
           "tcr_reduce_sum_exact_peer_emulated")


def tcr_reduce_sum_paper_f16(x, out, n=None, stream=None) -> None:
    """STUDY MODE: the paper's algorithm literally (fp16 everywhere, one launch per level)."""
    _check(_lib.tcr_reduce_sum_paper_f16(_ptr(x), _numel(x, n), _ptr(out), _stream(stream, x)),
           "tcr_reduce_sum_paper_f16")


def tcr_reduce_sum_study_fp32(x, out, kahan=False, n=None, stream=None) -> None:
    """STUDY MODE: the classic reduction entirely in binary32 (naive or Kahan)."""
    _check(_lib.tcr_reduce_sum_study_fp32(_ptr(x), _numel(x, n), 1 if kahan else 0, _ptr(out),
                                          _stream(stream, x)),
           "tcr_reduce_sum_study_fp32")


def tcr_probe_collapse(inp, out, algo=TCR_ALGO_MMA_SYNC, stream=None) -> None:
    """out[l] = lane l's result of the level-2 collapse of inp[0..32) (device float64)."""
    if isinstance(algo, str):
        algo = ALGOS[algo]
    _check(_lib.tcr_probe_collapse(_ptr(inp), _ptr(out), int(algo), _stream(stream, inp)),
           "tcr_probe_collapse")


def tcr_set_config(key: int, value: int) -> None:
    _check(_lib.tcr_set_config(int(key), int(value)), "tcr_set_config")


def tcr_get_config(key: int) -> int:
    return int(_lib.tcr_get_config(int(key)))


def tcr_launch_count() -> int:
    return int(_lib.tcr_launch_count())


def tcr_default_algo(n: int, dtype: int = TCR_DTYPE_F16) -> int:
    """The kernel TCR_ALGO_DEFAULT resolves to for n elements of dtype."""
    return int(_lib.tcr_default_algo(int(n), int(dtype)))


def tcr_release_workspaces() -> None:
    _check(_lib.tcr_release_workspaces(), "tcr_release_workspaces")


def tcr_version() -> int:
    return int(_lib.tcr_version())


def tcr_last_error() -> str:
    return _lib.tcr_last_error().decode()


def tcr_status_string(s: int) -> str:
    return _status_name(s)


# Convenience (allocating) wrappers --------------------------------------------------


def reduce_sum(x, algo: str | int = "default", exact: bool = False, out_dtype=None, stream=None):
    """Sum of a CUDA tensor (float16, bfloat16, float8_e4m3fn or float8_e5m2),
    returned as a 1-element device tensor (float32, or float64 with
    ``out_dtype=torch.float64``).  ``exact=True`` returns the correctly rounded
    exact sum (tcr_reduce_sum_exact_ex), for every supported type."""
    import torch

    x = x.reshape(-1) if x.is_contiguous() else x.contiguous().reshape(-1)
    f64 = out_dtype == torch.float64
    out = torch.empty(1, dtype=torch.float64 if f64 else torch.float32, device=x.device)
    if exact:
        tcr_reduce_sum_exact_ex(x, out_f32=None if f64 else out, out_f64=out if f64 else None,
                                stream=stream)
    else:
        tcr_reduce_sum_ex(x, out_f32=None if f64 else out, out_f64=out if f64 else None,
                          algo=algo, stream=stream)
    return out


def reduce_sum_segmented(x, offsets, mma: bool = True, stream=None):
    """Per-segment sums of a float16 / bfloat16 / float8 CUDA tensor over CSR int64 offsets."""
    import torch

    out = torch.empty(offsets.numel() - 1, dtype=torch.float32, device=x.device)
    tcr_reduce_sum_segmented_ex(x, offsets, out, algo="mma_sync" if mma else "shuffle",
                                stream=stream)
    return out


__all__ = [n for n in dir() if n.startswith("tcr_") or n.startswith("TCR_")] + [
    "reduce_sum", "reduce_sum_segmented", "TcrError", "LIB_PATH", "ALGOS"]
