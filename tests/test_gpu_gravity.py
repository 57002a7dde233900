"""GPU parity of the gravity slice (near-field monopole P2P behind the
reference's p2p_kernel launches, workload.cpp:365-372, 565-569) against the
oracle's orc_gravity_p2p: bitwise (the stencil table is geometry computed
with the same IEEE operations on both sides; per cell the same fma order)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("radius", [1, 2, 4, 6])
@pytest.mark.parametrize("periodic", ["", "xyz"])
def test_p2p_matches_oracle(hydro, oracle_lib, radius, periodic):
    m = hydro.uniform_mesh(4, 3, 4, periodic=periodic)
    dx = 1.0 / 32
    d = hydro.CudaDevice(hydro.HydroConfig(dx=dx))
    d.set_mesh(m)
    d.init_random(11)
    d.gravity_p2p(G=1.7, radius=radius)
    got = d.download_gravity()
    U = d.download()
    recs = [r for r in d.flush_activity() if r.name == "p2p_kernel"]
    d.close()
    want = oracle_lib.gravity_p2p(oracle_lib.params(nf=6, dx=dx), m.neighbor_ids, U, radius=radius, G=1.7)
    assert np.array_equal(got, want), f"max abs diff {np.abs(got - want).max():.3e}"
    assert len(recs) == 1


def test_p2p_per_subgrid_launches_on_many_streams(hydro, oracle_lib):
    """The reference schedule: one p2p launch per sub-grid on rotating
    streams after the step's hydro (here after a batched step); lists inline
    and run-split."""
    m = hydro.uniform_mesh(4, 4, 4)
    dx = 1.0 / 32
    d = hydro.CudaDevice(hydro.HydroConfig(dx=dx, n_species=2))
    d.set_mesh(m)
    d.init_random(3)
    d.step(1)
    fired = []
    for g in range(40):
        d.gravity_p2p(radius=4, owned_index=[g], stream_id=1 + g % 12, guid=g, done=lambda: fired.append(1))
    d.gravity_p2p(radius=4, owned_index=list(range(40, 64)), stream_id=5)
    got = d.download_gravity()
    U = d.download()
    d.close()
    assert len(fired) == 40
    want = oracle_lib.gravity_p2p(oracle_lib.params(nf=8, dx=dx), m.neighbor_ids, U, radius=4)
    assert np.array_equal(got, want)


def test_p2p_sedov_full_size_matches_oracle(hydro, oracle_lib):
    """BASELINE config 2's mesh (16^3 sub-grids): the density after 2 steps."""
    import os
    m = hydro.uniform_mesh(16, 16, 16)
    dx = 1.0 / 128
    d = hydro.CudaDevice(hydro.HydroConfig(dx=dx))
    d.set_mesh(m)
    U0 = hydro.ic_fill(d.config, "sedov", m, np.arange(m.n))
    d.upload(U0)
    d.step(2)
    d.gravity_p2p(radius=4)
    got = d.download_gravity()
    U = d.download()
    d.close()
    want = oracle_lib.gravity_p2p(oracle_lib.params(nf=6, dx=dx), m.neighbor_ids, U, radius=4)
    assert np.array_equal(got, want)


def test_p2p_contract_errors(hydro):
    d = hydro.CudaDevice(hydro.HydroConfig())
    d.set_mesh(hydro.uniform_mesh(2, 2, 2))
    with pytest.raises(ValueError, match="radius"):
        d.gravity_p2p(radius=7)
    with pytest.raises(hydro.TsError, match="no gravity"):
        d.download_gravity()
    d.close()
