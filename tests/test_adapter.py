"""The reference-side C++ adapter (include/ts_hydro_taskscope.hpp) built
against the reference's own headers and core (oracle/_ref, compiled in the
build container): links on CPU; on a GPU its CompletionTokens fulfil and the
reference Profiler receives the kernels' ActivityRecords."""
import os
import subprocess

import pytest

from tests.conftest import ROOT

ADAPTER = os.path.join(ROOT, "oracle", "_ref", "adapter_check")


def _need():
    if not os.path.exists(ADAPTER):
        pytest.skip("oracle/_ref/adapter_check not built (needs /root/reference at build time)")


def test_adapter_links_against_reference_core():
    _need()
    r = subprocess.run([ADAPTER], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and "adapter links" in r.stdout


@pytest.mark.gpu
def test_adapter_feeds_reference_profiler_on_gpu():
    _need()
    r = subprocess.run([ADAPTER, "run"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "hydro_stage1_kernel calls 8" in r.stdout
