import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")
    # A fresh checkout has no built libraries (they are git-ignored): build
    # them once (nvcc cross-compiles for sm_100a without a GPU).
    libs = (os.path.join(ROOT, "paper_1903_03640_b200", "libtcr.so"),
            os.path.join(ROOT, "tcr_inputs", "libtcr_inputs.so"))
    if not all(os.path.exists(p) for p in libs):
        import __graft_entry__

        __graft_entry__.build()


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def paper_golden():
    return load_golden("paper_model.json")


@pytest.fixture(scope="session")
def spec_golden():
    return load_golden("spec_examples.json")
