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


@pytest.fixture(autouse=True)
def _self_check_build_clean():
    """With TS_HYDRO_CHECK_STRICT=1 and a TS_CHECK library (TS_HYDRO_LIB), every
    device a test closed or dropped must have recorded no protocol / bounds
    failure (the stand-in for compute-sanitizer)."""
    yield
    if not os.environ.get("TS_HYDRO_CHECK_STRICT"):
        return
    import gc
    from paper_2210_06437_b200 import hydro as H
    gc.collect()
    bad = list(H.CHECK_FAILURES)
    H.CHECK_FAILURES.clear()
    assert not bad, f"self-check failures recorded: {bad}"
