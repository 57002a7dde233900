"""GPU parity of the gravity FMM (the reference's
multipole_root / multipole / p2m / p2p launches, workload.cpp:365-372) against
the oracle's orc_gravity_fmm: bitwise — the kernels follow the oracle
operation for operation (IEEE sqrt and division, explicit fma, --fmad=false),
on uniform meshes (power-of-two and not), coarse-fine AMR meshes, the
reference's own build_mesh octrees and a lone root sub-grid."""
import numpy as np
import pytest

from paper_2210_06437_b200 import amr

pytestmark = pytest.mark.gpu

L_SHAPE = {(0, 1, 1, 1), (0, 2, 1, 1), (0, 1, 2, 1), (0, 1, 1, 2), (0, 2, 2, 2)}


def blob(level, pos, dx0, nf, centre=(0.55, 0.45, 0.5), width=0.2, seed=0):
    """A smooth density blob plus a little noise (so every cell differs)."""
    rng = np.random.default_rng(seed)
    U = np.zeros((len(level), nf, 512))
    i = np.arange(512)
    loc = np.stack([i & 7, (i >> 3) & 7, i >> 6]).astype(float)
    for k in range(len(level)):
        h = dx0 * 2.0 ** -int(level[k])
        xc = (np.asarray(pos[k], float)[:, None] * 8 + loc + 0.5) * h
        r2 = ((xc - np.asarray(centre)[:, None]) ** 2).sum(0)
        U[k, 0] = np.exp(-r2 / width ** 2) + 0.01 + 0.001 * rng.random(512)
        U[k, 4] = 1.0
    return U


def fmm_gpu(hydro, setup, U, radius, G=1.3, dx=1.0 / 32, **kw):
    d = hydro.CudaDevice(hydro.HydroConfig(dx=dx, **kw))
    setup(d)
    d.upload(U)
    d.set_gravity_tree()
    d.gravity_fmm(G=G, radius=radius)
    got = d.download_gravity()
    recs = d.flush_activity()
    d.close()
    return got, recs


@pytest.mark.parametrize("radius", [1, 2, 3])
@pytest.mark.parametrize("dims", [(4, 4, 4), (3, 2, 5)])
def test_fmm_uniform_matches_oracle(hydro, oracle_lib, radius, dims):
    m = hydro.uniform_mesh(*dims)
    dx = 1.0 / 32
    lev = np.zeros(m.n, np.int32)
    U = blob(lev, m.pos, dx, 6)
    got, recs = fmm_gpu(hydro, lambda d: d.set_mesh(m), U, radius, dx=dx)
    want = oracle_lib.gravity_fmm(6, lev, m.pos, m.dims, dx, U, radius=radius, G=1.3)
    assert np.array_equal(got, want), f"max abs diff {np.abs(got - want).max():.3e}"
    names = {r.name for r in recs}
    assert {"fmm_moments_kernel", "multipole_root_kernel", "p2p_kernel"} <= names


@pytest.mark.parametrize("radius", [2, 3])
def test_fmm_amr_matches_oracle(hydro, oracle_lib, radius):
    m = amr.amr_mesh(4, 4, 4, L_SHAPE)
    dx = 1.0 / 64  # finest level
    dx0 = dx * 2
    U = blob(m.level, m.pos, dx0, 7)
    got, recs = fmm_gpu(hydro, lambda d: d.set_amr_mesh(m), U, radius, dx=dx, n_species=1)
    want = oracle_lib.gravity_fmm(7, m.level, m.pos, m.dims, dx0, U, radius=radius, G=1.3)
    assert np.array_equal(got, want), f"max abs diff {np.abs(got - want).max():.3e}"
    names = [r.name for r in recs]
    assert "p2m_kernel" in names and "multipole_kernel" in names


def test_fmm_reference_octrees_match_oracle(hydro, oracle_lib, golden):
    """The reference's own build_mesh octrees (root = one sub-grid, 3 and 4 levels)."""
    vec, _ = golden
    for mm in vec["build_mesh"]:
        if mm["levels"] < 3:
            continue
        a = amr.from_reference_mesh(mm["level"], mm["pos"])
        dx = 1.0 / (8 << a.max_level)
        dx0 = 1.0 / 8
        U = blob(a.level, a.pos, dx0, 6, centre=(0.4, 0.55, 0.5), width=0.25)
        got, _ = fmm_gpu(hydro, lambda d: d.set_amr_mesh(a), U, 2, dx=dx)
        want = oracle_lib.gravity_fmm(6, a.level, a.pos, a.dims, dx0, U, radius=2, G=1.3)
        assert np.array_equal(got, want), f"levels={mm['levels']}: max abs diff {np.abs(got - want).max():.3e}"


def test_fmm_single_subgrid_root_leaf(hydro, oracle_lib):
    m = hydro.uniform_mesh(1, 1, 1)
    dx = 1.0 / 8
    lev = np.zeros(1, np.int32)
    U = blob(lev, m.pos, dx, 6, centre=(0.5, 0.5, 0.5))
    got, recs = fmm_gpu(hydro, lambda d: d.set_mesh(m), U, 2, dx=dx)
    want = oracle_lib.gravity_fmm(6, lev, m.pos, m.dims, dx, U, radius=2, G=1.3)
    assert np.array_equal(got, want)
    direct = oracle_lib.gravity_direct(6, lev, m.pos, m.dims, dx, U, G=1.3)
    assert np.allclose(got, direct, rtol=1e-12, atol=0)
    assert [r.name for r in recs if r.name.endswith("_kernel")] == ["fmm_moments_kernel", "multipole_root_kernel"]


def test_fmm_after_steps_sedov_8cubed(hydro, oracle_lib):
    """The state after two hydro steps (8^3 sub-grids, Sedov), row-ordered
    mesh: the tree follows the positions, not the storage order."""
    m = hydro.uniform_mesh(8, 8, 8, order="row")
    dx = 1.0 / 64
    d = hydro.CudaDevice(hydro.HydroConfig(dx=dx))
    d.set_mesh(m)
    d.upload(hydro.ic_fill(d.config, "sedov", m, np.arange(m.n)))
    d.step(2)
    d.set_gravity_tree()
    d.gravity_fmm(G=1.0, radius=2)
    got = d.download_gravity()
    U = d.download()
    d.close()
    want = oracle_lib.gravity_fmm(6, np.zeros(m.n, np.int32), m.pos, m.dims, dx, U, radius=2, G=1.0)
    assert np.array_equal(got, want)


def test_fmm_refusals(hydro):
    m = hydro.uniform_mesh(2, 2, 2)
    d = hydro.CudaDevice(hydro.HydroConfig(dx=1.0 / 16))
    d.set_mesh(m)
    d.init_random(1)
    with pytest.raises(Exception, match="gravity tree"):
        d.gravity_fmm()
    with pytest.raises(ValueError):
        d.set_gravity_tree(np.zeros(8, np.int32), np.zeros((8, 3), np.int32), (2, 2, 2), 1.0 / 16)  # duplicates
    d.set_gravity_tree()
    with pytest.raises(ValueError):
        d.gravity_fmm(radius=4)
    d.close()


def test_fmm_one_context_every_radius_twice(hydro, oracle_lib):
    """One context, radii 3, 1, 2, 3 back to back (the tables of every radius
    live side by side; the set-up copies have landed before the first solve)."""
    m = hydro.uniform_mesh(4, 4, 2)
    dx = 1.0 / 32
    lev = np.zeros(m.n, np.int32)
    U = blob(lev, m.pos, dx, 6, seed=5)
    d = hydro.CudaDevice(hydro.HydroConfig(dx=dx))
    d.set_mesh(m)
    d.upload(U)
    d.set_gravity_tree()
    for R in (3, 1, 2, 3):
        d.gravity_fmm(G=0.7, radius=R)
        got = d.download_gravity()
        want = oracle_lib.gravity_fmm(6, lev, m.pos, m.dims, dx, U, radius=R, G=0.7)
        assert np.array_equal(got, want), R
    d.close()


def test_gravity_kick_matches_oracle(hydro, oracle_lib):
    m = hydro.uniform_mesh(4, 2, 2)
    dx = 1.0 / 32
    lev = np.zeros(m.n, np.int32)
    d = hydro.CudaDevice(hydro.HydroConfig(dx=dx, n_species=2))
    d.set_mesh(m)
    d.init_random(9)
    U0 = d.download()
    d.set_gravity_tree()
    d.gravity_fmm(G=2.0, radius=2)
    g = d.download_gravity()
    d.gravity_kick(1e-3)
    got = d.download()
    recs = [r.name for r in d.flush_activity()]
    d.close()
    want = oracle_lib.gravity_kick(U0, g, 1e-3)
    assert np.array_equal(got, want)
    assert "gravity_kick_kernel" in recs


@pytest.mark.parametrize("case", ["uniform", "amr"])
def test_step_gravity_matches_oracle(hydro, oracle_lib, case):
    """Hydro + self-gravity on the device (step, FMM, kick per step; dt from
    the kicked state) against the oracle's same loop: bitwise, equal dts."""
    if case == "uniform":
        m = hydro.uniform_mesh(4, 4, 4)
        dx = 1.0 / 32
        level, pos, dims, dx0 = np.zeros(m.n, np.int32), m.pos, m.dims, dx
        U0 = blob(level, pos, dx0, 6, centre=(0.5, 0.5, 0.5), width=0.15)
        setup = lambda d: d.set_mesh(m)  # noqa: E731
        nbr, mesh = m.neighbor_ids, None
    else:
        mesh = amr.amr_mesh(4, 4, 4, L_SHAPE)
        dx = 1.0 / 64
        level, pos, dims, dx0 = mesh.level, mesh.pos, mesh.dims, 2 * dx
        U0 = blob(level, pos, dx0, 6, centre=(0.4, 0.45, 0.5), width=0.15)
        setup = lambda d: d.set_amr_mesh(mesh)  # noqa: E731
        nbr = None
    U0[:, 4] = 0.05 + 0.5 * U0[:, 0]  # warm, at rest
    d = hydro.CudaDevice(hydro.HydroConfig(dx=dx))
    setup(d)
    d.upload(U0)
    d.set_gravity_tree()
    d.step_gravity(3, G=3.0, radius=2)
    got = d.download()
    dt = d.last_dt()
    d.close()
    want, dts = oracle_lib.run_self_gravity(oracle_lib.params(nf=6, dx=dx), nbr, U0, 3, level, pos, dims, dx0,
                                            radius=2, G=3.0, mesh=mesh)
    assert dt == dts[-1]
    assert np.array_equal(got, want), f"max abs diff {np.abs(got - want).max():.3e}"


def test_fmm_full_size_sedov_and_amr_match_oracle(hydro, oracle_lib):
    """BASELINE config 2's mesh (16^3 sub-grids, 2 M cells) after two Sedov
    steps, and a 16^3 AMR mesh with a refined centre (4544 leaves): bitwise."""
    m = hydro.uniform_mesh(16, 16, 16, order="row")
    dx = 1.0 / 128
    d = hydro.CudaDevice(hydro.HydroConfig(dx=dx))
    d.set_mesh(m)
    d.upload(hydro.ic_fill(d.config, "sedov", m, np.arange(m.n)))
    d.step(2)
    d.set_gravity_tree()
    d.gravity_fmm(G=1.0, radius=2)
    got = d.download_gravity()
    U = d.download()
    d.close()
    want = oracle_lib.gravity_fmm(6, np.zeros(m.n, np.int32), m.pos, m.dims, dx, U, radius=2, G=1.0)
    assert np.array_equal(got, want)
    a = amr.amr_mesh(16, 16, 16, lambda L, p: all(6 <= v < 10 for v in p))
    dx = 1.0 / 256
    U0 = blob(a.level, a.pos, 2 * dx, 6, centre=(0.5, 0.5, 0.5), width=0.1)
    got, recs = fmm_gpu(hydro, lambda d: d.set_amr_mesh(a), U0, 2, dx=dx)
    want = oracle_lib.gravity_fmm(6, a.level, a.pos, a.dims, 2 * dx, U0, radius=2, G=1.3)
    assert np.array_equal(got, want)
    assert {"p2p_kernel", "p2m_kernel", "multipole_kernel", "multipole_root_kernel"} <= {r.name for r in recs}


def test_gravity_on_another_stream_is_ordered_before_the_next_step(hydro, oracle_lib):
    """A solve issued on stream 7 reads U^n; the step issued right after it on
    the compute stream rewrites U^n in stage 3 — it must wait for the solve
    (the join of the gravity streams), so the field is the pre-step state's."""
    m = hydro.uniform_mesh(16, 16, 16, order="row")
    dx = 1.0 / 128
    d = hydro.CudaDevice(hydro.HydroConfig(dx=dx))
    d.set_mesh(m)
    d.upload(hydro.ic_fill(d.config, "sedov", m, np.arange(m.n)))
    d.step(1)
    U = d.download()
    d.set_gravity_tree()
    d.gravity_fmm(G=1.0, radius=2, stream_id=7)
    d.step(1)  # no host wait in between
    got = d.download_gravity()
    d.close()
    want = oracle_lib.gravity_fmm(6, np.zeros(m.n, np.int32), m.pos, m.dims, dx, U, radius=2, G=1.0)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("merge", ["0", "1"])
@pytest.mark.parametrize("radius", [1, 3])
def test_fmm_merged_and_per_depth_m2l_match_oracle(hydro, oracle_lib, monkeypatch, merge, radius):
    """The M2L part sums of the root and the depths below it as ONE launch
    (default; R = 3 merges only the depths that fit the scratch) or one launch
    per depth (TS_HYDRO_FMM_MERGE=0): both bitwise to the oracle, on an 8^3
    mesh (refined depths 0-2, so the merge spans two depths below the root)."""
    monkeypatch.setenv("TS_HYDRO_FMM_MERGE", merge)
    m = hydro.uniform_mesh(8, 8, 8)
    dx = 1.0 / 64
    lev = np.zeros(m.n, np.int32)
    U = blob(lev, m.pos, dx, 6)
    got, _ = fmm_gpu(hydro, lambda d: d.set_mesh(m), U, radius, dx=dx)
    want = oracle_lib.gravity_fmm(6, lev, m.pos, m.dims, dx, U, radius=radius, G=1.3)
    assert np.array_equal(got, want), f"max abs diff {np.abs(got - want).max():.3e}"
