"""The C ABI from plain C: examples/c_api_demo.c builds against include/tcr.h
and libtcr.so with gcc (CPU), and runs correctly on a B200 (GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_demo_builds():
    import __graft_entry__ as g

    exe = g.build_c_demo()
    assert os.access(exe, os.X_OK)


@pytest.mark.gpu
def test_c_demo_runs():
    import __graft_entry__ as g

    exe = g.build_c_demo()
    for n in ("1", "1000", str((1 << 24) + 3)):
        r = subprocess.run([exe, n], capture_output=True, text=True, timeout=120)
        assert r.returncode == 0, r.stdout + r.stderr
        assert "OK" in r.stdout
