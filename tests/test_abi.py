"""CPU-side checks of the C-ABI library: it loads, exports every symbol that
include/tcr.h declares, and its host-side validation answers without touching
a device.  (No compute calls: there is no GPU in this container.)"""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tcr.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(tcr_[a-z0-9_]+)\s*\(", src))
    assert len(names) >= 15
    return sorted(names)


def test_header_symbols_exported():
    import paper_1903_03640_b200 as tcr

    lib = ctypes.CDLL(tcr.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), f"{name} declared in tcr.h but not exported"


def test_binding_names_match_abi():
    import paper_1903_03640_b200 as tcr

    for name in declared_symbols():
        if name in ("tcr_status_string", "tcr_last_error"):
            continue
        assert hasattr(tcr, name), f"python binding lacks {name}"


def test_version_and_status_strings():
    import paper_1903_03640_b200 as tcr

    assert tcr.tcr_version() == 100
    assert tcr.tcr_status_string(0) == "TCR_OK"
    assert tcr.tcr_status_string(2) == "TCR_ERR_UNSUPPORTED_DEVICE"
    assert tcr.tcr_launch_count() >= 0


def test_invalid_arguments_rejected_before_device():
    import paper_1903_03640_b200 as tcr

    with pytest.raises(tcr.TcrError) as e:
        tcr.tcr_reduce_sum(0, 0, n=16, stream=0)  # x NULL with n > 0
    assert e.value.status == tcr.TCR_ERR_INVALID_VALUE
    with pytest.raises(tcr.TcrError) as e:
        tcr.tcr_reduce_sum(0x1001, 0x2000, n=16, stream=0)  # x not 2-byte aligned
    assert e.value.status == tcr.TCR_ERR_INVALID_VALUE
    with pytest.raises(tcr.TcrError) as e:
        tcr.tcr_reduce_sum_algo(0x1000, 0x2000, None, algo=99, n=16, stream=0)
    assert e.value.status == tcr.TCR_ERR_INVALID_VALUE
    with pytest.raises(tcr.TcrError) as e:
        tcr.tcr_reduce_sum_segmented(0x1000, 0, 0x2000, num_segments=4, stream=0)
    assert e.value.status == tcr.TCR_ERR_INVALID_VALUE
    # fused peer combine: group shape, algo and mailboxes are checked first
    mb = [0x10000 + 0x1000 * r for r in range(9)]
    F16 = tcr.TCR_DTYPE_F16
    for args in ((mb[:9], 0, 1), (mb[:0], 0, 1), (mb[:2], 2, 1), (mb[:2], -1, 1),
                 (mb[:2], 0, tcr.TCR_ALGO_BULK_MMA), ([0x10000, 0], 0, 1), ([0x10008], 0, 1)):
        with pytest.raises(tcr.TcrError) as e:
            tcr.tcr_reduce_sum_peer(0x1000, args[0], args[1], out_f32=0x2000, algo=args[2],
                                    dtype=F16, n=16, stream=0)
        assert e.value.status == tcr.TCR_ERR_INVALID_VALUE, args
    with pytest.raises(tcr.TcrError) as e:
        tcr.tcr_reduce_sum_peer_emulated(0x1000, mb[:2], algo=1, dtype=F16, n=16, stream=0)
    assert e.value.status == tcr.TCR_ERR_INVALID_VALUE  # no output
    for args in ((mb[:9], 0), (mb[:2], 5), ([0x10000, 0], 0)):
        with pytest.raises(tcr.TcrError) as e:
            tcr.tcr_reduce_sum_exact_peer(0x1000, args[0], args[1], out_f32=0x2000, n=16, stream=0)
        assert e.value.status == tcr.TCR_ERR_INVALID_VALUE, args
    with pytest.raises(tcr.TcrError) as e:  # no output at all
        tcr.tcr_reduce_sum_exact_peer_emulated(0x1000, mb[:2], n=16, stream=0)
    assert e.value.status == tcr.TCR_ERR_INVALID_VALUE
    with pytest.raises(ValueError):
        tcr.tcr_peer_ipc_open(b"short")


def test_config_validation():
    import paper_1903_03640_b200 as tcr

    old = tcr.tcr_get_config(tcr.TCR_CFG_UNROLL)
    with pytest.raises(tcr.TcrError):
        tcr.tcr_set_config(tcr.TCR_CFG_UNROLL, 5)
    tcr.tcr_set_config(tcr.TCR_CFG_UNROLL, 16)
    assert tcr.tcr_get_config(tcr.TCR_CFG_UNROLL) == 16
    tcr.tcr_set_config(tcr.TCR_CFG_UNROLL, old)
    with pytest.raises(tcr.TcrError):
        tcr.tcr_set_config(tcr.TCR_CFG_TC05_STAGE_KB, 6)
    assert tcr.tcr_get_config(99) == -1
    assert tcr.tcr_get_config(tcr.TCR_CFG_PDL) == 1  # programmatic dependent launch on by default
    with pytest.raises(tcr.TcrError):
        tcr.tcr_set_config(tcr.TCR_CFG_PDL, 2)


def test_product_path_does_not_import_oracle():
    # The product package must not reference the test oracle (independence rule).
    pkg = os.path.join(ROOT, "paper_1903_03640_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in src.replace("oracle/", ""), f


def test_sass_is_sm100a_with_tensor_core_instructions():
    # cuobjdump runs on the host: the library carries sm_100a SASS with the
    # legacy tensor path (HMMA/DMMA) and the tcgen05 path (UTCHMMA, LDTM, UBLKCP).
    import shutil
    import subprocess

    import paper_1903_03640_b200 as tcr

    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run(["cuobjdump", "-sass", tcr.LIB_PATH], capture_output=True,
                          text=True, check=True).stdout
    assert "sm_100a" in sass
    for mnemonic in ("HMMA.16816.F32", "DMMA.8x8x4", "UTCHMMA", "LDTM", "UBLKCP"):
        assert mnemonic in sass, mnemonic


def test_sass_fused_peer_kernel_has_mma_and_system_scope_peer_traffic():
    """NEXT-2 evidence in SASS: the fused kernel (reduce_stream_kernel<..., kPeer
    = true>) carries the tensor-core tiles (HMMA), the level-2 DMMA collapse,
    the 16-byte system-scope stores of the push (STG.E.128.STRONG.SYS, to the
    peers' mapped mailboxes), the system-scope polls and the %globaltimer
    bound -- one kernel, no separate collective."""
    import re
    import shutil
    import subprocess

    import paper_1903_03640_b200 as tcr

    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run(["cuobjdump", "-sass", tcr.LIB_PATH], capture_output=True,
                          text=True, check=True).stdout
    funcs = re.split(r"\n\s+Function : ", sass)[1:]
    peer = [f for f in funcs if f.startswith("_ZN3tcr20reduce_stream_kernelILb1ELi0ELi4ELi8ELb1E")]
    assert peer, "fused peer kernel not found"
    body = peer[0]
    for mnemonic in ("HMMA.16816.F32", "DMMA.8x8x4", "STG.E.128.STRONG.SYS", "LDG.E.128.STRONG.SYS",
                     "SR_GLOBALTIMER", "NANOSLEEP"):
        assert mnemonic in body, mnemonic
    plain = [f for f in funcs if f.startswith("_ZN3tcr20reduce_stream_kernelILb1ELi0ELi4ELi8ELb0E")]
    assert plain and "STRONG.SYS" not in plain[0]  # the plain kernel has no peer traffic
    # r02: the same combine fused into the tcgen05 kernel (tight loop, KM = 8):
    # UTCHMMA tiles from SMEM + the DMMA collapse + the system-scope push / poll
    tpeer = [f for f in funcs if f.startswith("_ZN3tcr21reduce_tcgen05_kernelILb0ELi8ELb1E")]
    assert tpeer, "fused tcgen05 peer kernel not found"
    for mnemonic in ("UTCHMMA", "UBLKCP", "LDTM", "DMMA.8x8x4", "STG.E.128.STRONG.SYS",
                     "LDG.E.128.STRONG.SYS"):
        assert mnemonic in tpeer[0], mnemonic
    tplain = [f for f in funcs if f.startswith("_ZN3tcr21reduce_tcgen05_kernelILb0ELi8ELb0E")]
    assert tplain and "STRONG.SYS" not in tplain[0]


def test_sass_dynamic_tail_and_rows_kernels():
    """r02 §16-§17 in SASS: the default large-n kernel (tcgen05 with the
    dynamic tail) carries the bulk copies into SMEM (UBLKCP), the tensor-core
    tiles (UTCHMMA), the TMEM reads (LDTM), the per-round D' = 1 x D DMMA
    collapse and the chunk-ticket atomics; the batched rows kernel loads its
    boxes with 2-D TMA tensor copies (UTMALDG.2D) and reduces them with
    UTCHMMA."""
    import re
    import shutil
    import subprocess

    import paper_1903_03640_b200 as tcr

    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run(["cuobjdump", "-sass", tcr.LIB_PATH], capture_output=True,
                          text=True, check=True).stdout
    funcs = re.split(r"\n\s+Function : ", sass)[1:]
    dyn = [f for f in funcs if f.startswith("_ZN3tcr21reduce_tcgen05_kernelILb0ELi8ELb0ELb1E")]
    assert dyn, "dynamic-tail tcgen05 kernel not found"
    for mnemonic in ("UBLKCP", "UTCHMMA", "LDTM", "DMMA.8x8x4", "ATOMG"):
        assert mnemonic in dyn[0], mnemonic
    rows = [f for f in funcs if "reduce_rows_tc05_kernel" in f.split("\n", 1)[0]]
    assert rows, "tcgen05 rows kernel not found"
    for mnemonic in ("UTMALDG.2D", "UTCHMMA", "LDTM"):
        assert mnemonic in rows[0], mnemonic


def test_product_path_fails_loudly_without_the_library(tmp_path):
    """No fallback: a copy of the package without libtcr.so refuses to import."""
    import shutil
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pkg = os.path.join(root, "paper_1903_03640_b200")
    dst = tmp_path / "paper_1903_03640_b200"
    shutil.copytree(pkg, dst, ignore=shutil.ignore_patterns("*.so", "csrc", "__pycache__"))
    r = subprocess.run([sys.executable, "-c", "import paper_1903_03640_b200"], cwd=tmp_path,
                       capture_output=True, text=True, env={**os.environ, "PYTHONPATH": str(tmp_path)})
    assert r.returncode != 0
    assert "ImportError" in r.stderr and "no fallback" in r.stderr


def test_no_register_spills_in_any_kernel():
    """Every kernel of libtcr.so compiles without register spills (ptxas -v
    report written by the Makefile next to each object; r02)."""
    import subprocess

    csrc = os.path.join(ROOT, "paper_1903_03640_b200", "csrc")
    subprocess.run(["make", "-s", "-C", csrc], check=True, capture_output=True)
    objdir = os.path.join(ROOT, "build", "obj")
    reports = [f for f in os.listdir(objdir) if f.endswith(".ptxas.txt")]
    assert len(reports) >= 8
    seen, bad = 0, []
    for f in reports:
        for blk in open(os.path.join(objdir, f)).read().split("Compiling entry function '")[1:]:
            name = blk.split("'")[0]
            m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", blk)
            if m:
                seen += 1
                if int(m.group(1)) or int(m.group(2)):
                    bad.append((f, name, m.group(0)))
    assert seen >= 50, seen
    assert not bad, bad[:5]


def test_round2_knobs_defaults_and_ranges():
    """r02 §16-§18 knobs: defaults, accepted ranges, rejected values restore
    nothing.  Host logic only (no device work)."""
    import paper_1903_03640_b200 as tcr

    cases = [  # (key, default, accepted, rejected)
        (tcr.TCR_CFG_TC05_DYNAMIC, 8, (0, 100), (-1, 101)),
        (tcr.TCR_CFG_TC05_DYN_MIN_RUN, 32, (0, 1 << 20), (-1, (1 << 20) + 1)),
        (tcr.TCR_CFG_ROWS_TC05, 1, (0, 1), (2, -1)),
        (tcr.TCR_CFG_ROWS_TC05_STAGES, 4, (2, 6), (1, 7)),
        (tcr.TCR_CFG_EXACT_BULK, 1, (0, 2), (3, -1)),
    ]
    for key, default, ok, bad in cases:
        assert tcr.tcr_get_config(key) == default, key
        try:
            for v in ok:
                tcr.tcr_set_config(key, v)
                assert tcr.tcr_get_config(key) == v
            tcr.tcr_set_config(key, default)
            for v in bad:
                with pytest.raises(tcr.TcrError):
                    tcr.tcr_set_config(key, v)
                assert tcr.tcr_get_config(key) == default
        finally:
            tcr.tcr_set_config(key, default)


def test_default_algo_resolution():
    """TCR_ALGO_DEFAULT resolves to TCR_CFG_DEFAULT_ALGO; its default, 0 = auto,
    picks by input size and format (r02 §16): tcgen05 (dynamic tail) for
    binary16 and fp8 from 512 MiB, mma.sync below and for bfloat16 at every
    size.  Host logic only (no device work)."""
    import paper_1903_03640_b200 as tcr

    assert tcr.tcr_get_config(tcr.TCR_CFG_DEFAULT_ALGO) == tcr.TCR_ALGO_DEFAULT
    assert tcr.tcr_get_config(tcr.TCR_CFG_TC05_DYNAMIC) == 8
    assert tcr.tcr_get_config(tcr.TCR_CFG_TC05_DYN_MIN_RUN) == 32
    f16, bf16, e4, e5 = tcr.TCR_DTYPE_F16, tcr.TCR_DTYPE_BF16, tcr.TCR_DTYPE_E4M3, tcr.TCR_DTYPE_E5M2
    assert tcr.tcr_default_algo(1 << 16, f16) == tcr.TCR_ALGO_MMA_SYNC
    assert tcr.tcr_default_algo((1 << 28) - 1, f16) == tcr.TCR_ALGO_MMA_SYNC
    assert tcr.tcr_default_algo(1 << 28, f16) == tcr.TCR_ALGO_TCGEN05  # 512 MiB
    assert tcr.tcr_default_algo(1 << 30, f16) == tcr.TCR_ALGO_TCGEN05  # C3
    for n in (1 << 16, 1 << 30, 1 << 33):
        assert tcr.tcr_default_algo(n, bf16) == tcr.TCR_ALGO_MMA_SYNC
    for fmt in (e4, e5):
        assert tcr.tcr_default_algo((1 << 29) - 1, fmt) == tcr.TCR_ALGO_MMA_SYNC
        assert tcr.tcr_default_algo(1 << 29, fmt) == tcr.TCR_ALGO_TCGEN05
    try:
        tcr.tcr_set_config(tcr.TCR_CFG_DEFAULT_ALGO, tcr.TCR_ALGO_MMA_SYNC)
        for n in (1 << 16, 1 << 29, 1 << 33):
            assert tcr.tcr_default_algo(n, f16) == tcr.TCR_ALGO_MMA_SYNC
        tcr.tcr_set_config(tcr.TCR_CFG_DEFAULT_ALGO, tcr.TCR_ALGO_SHUFFLE)
        assert tcr.tcr_default_algo(1 << 31, f16) == tcr.TCR_ALGO_SHUFFLE
    finally:
        tcr.tcr_set_config(tcr.TCR_CFG_DEFAULT_ALGO, tcr.TCR_ALGO_DEFAULT)
