import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    # the C-ABI library is a build artefact (git-ignored): build it in-tree if
    # a fresh checkout runs the tests before __graft_entry__.build()
    lib = os.path.join(ROOT, "paper_1701_03787_b200", "libshen_b200.so")
    if not os.path.exists(lib):
        import subprocess

        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_1701_03787_b200", "csrc"), "-j8"], check=False)


def _gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _gpu_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(os.path.join(GOLDEN, name))
    return load


@pytest.fixture(scope="session")
def golden_meta():
    with open(os.path.join(GOLDEN, "golden_meta.json")) as fh:
        return json.load(fh)
