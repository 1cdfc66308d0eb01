import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")


def _have_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _have_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    import json

    def load(name):
        with open(os.path.join(ROOT, "tests", "golden", name)) as f:
            return json.load(f)
    return load


@pytest.fixture(scope="session")
def coracle():
    import oracle_py
    oracle_py.build()
    return oracle_py.COracle()


@pytest.fixture(scope="session")
def mesh1d():
    """The reference's 1D mesh hierarchies (tests/golden/mesh1d, written by
    oracle/make_golden.py --only-mesh1d from its build_hierarchy) as
    wavemc.Mesh1D lists: mesh1d(name, max_level=4)."""
    import json

    def load(name, max_level=4):
        from paper_2106_11117_b200 import wavemc
        with open(os.path.join(ROOT, "tests", "golden", "mesh1d", f"{name}_L4.json")) as f:
            h = json.load(f)
        return wavemc.Mesh1D.hierarchy(h["levels"][: max_level + 1])
    return load
