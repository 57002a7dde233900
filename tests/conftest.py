"""Shared pytest setup.

Markers: `gpu` tests need a B200 (run with `-m gpu` on the GPU box); every
other test runs on CPU in a few minutes.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")
    config.addinivalue_line("markers", "slow: longer CPU test")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def hydro():
    from paper_2210_06437_b200 import hydro as H
    if not os.path.exists(H.LIB_PATH):
        from paper_2210_06437_b200 import build
        build.build()
    H.lib()
    return H


@pytest.fixture(scope="session")
def golden():
    import json
    import numpy as np
    d = os.path.join(ROOT, "tests", "golden")
    with open(os.path.join(d, "reference_vectors.json")) as f:
        vec = json.load(f)
    ghosts = dict(np.load(os.path.join(d, "reference_ghosts.npz")))
    return vec, ghosts
