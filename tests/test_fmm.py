"""The gravity FMM oracle (oracle/fmm_oracle.c) on the CPU:
accuracy against a brute-force pair sum, convergence with the interaction
radius, the interaction tables, malformed trees.  The GPU is held to this
oracle bitwise (tests/test_gpu_fmm.py)."""
import numpy as np
import pytest

from paper_2210_06437_b200 import amr


def blob(level, pos, dx0, nf=6, centre=(0.55, 0.45, 0.5), width=0.2):
    U = np.zeros((len(level), nf, 512))
    i = np.arange(512)
    loc = np.stack([i & 7, (i >> 3) & 7, i >> 6]).astype(float)
    for k in range(len(level)):
        h = dx0 * 2.0 ** -int(level[k])
        xc = (np.asarray(pos[k], float)[:, None] * 8 + loc + 0.5) * h
        U[k, 0] = np.exp(-((xc - np.asarray(centre)[:, None]) ** 2).sum(0) / width ** 2) + 0.01
    return U


def errors(oracle_lib, level, pos, dims, dx0, R):
    U = blob(level, pos, dx0)
    f = oracle_lib.gravity_fmm(6, level, pos, dims, dx0, U, radius=R)
    d = oracle_lib.gravity_direct(6, level, pos, dims, dx0, U)
    ephi = np.abs(f[:, 0] - d[:, 0]).max() / np.abs(d[:, 0]).max()
    gmag = np.sqrt((d[:, 1:] ** 2).sum(1))
    eg = np.sqrt(((f[:, 1:] - d[:, 1:]) ** 2).sum(1)).max() / gmag.max()
    return ephi, eg


def grid_positions(nx, ny, nz):
    return np.array([[x, y, z] for z in range(nz) for y in range(ny) for x in range(nx)], np.int32)


def test_fmm_tables(oracle_lib):
    sizes = {R: len(oracle_lib.fmm_table(R)[0]) for R in (1, 2, 3)}
    assert sizes == {1: 55, 2: 263, 3: 983}
    u, near = oracle_lib.fmm_table(2)
    r2 = (u ** 2).sum(1)
    assert near.sum() == 32 and np.array_equal(near, r2 <= 4)
    # the octant-0 table mirrored is every other octant's interaction set (the
    # GPU reads mirrored offsets): e in the set of a cell of parity p iff its
    # parent offset ((p + e) >> 1) - (p >> 1) lies within R
    for px in (0, 1):
        for py in (0, 1):
            for pz in (0, 1):
                p = np.array([px, py, pz])
                sig = np.where(p == 1, -1, 1)
                mirrored = {tuple(sig * v) for v in u}
                K = 5
                rng = np.arange(-K, K + 1)
                e = np.stack(np.meshgrid(rng, rng, rng, indexing="ij"), -1).reshape(-1, 3)
                par = ((p + e) >> 1) - (p >> 1)
                member = ((par ** 2).sum(1) <= 4) & (np.abs(e).sum(1) > 0)
                assert mirrored == {tuple(v) for v in e[member]}
    ur, _ = oracle_lib.fmm_table(2, root=True)
    assert len(ur) == 15 ** 3 - 1


@pytest.mark.parametrize("R,phi_tol,g_tol", [(1, 6e-3, 0.12), (2, 2e-3, 0.04), (3, 8e-4, 0.02)])
def test_fmm_accuracy_uniform(oracle_lib, R, phi_tol, g_tol):
    pos = grid_positions(2, 2, 2)
    ephi, eg = errors(oracle_lib, np.zeros(8, np.int32), pos, (2, 2, 2), 1.0 / 16, R)
    assert ephi < phi_tol and eg < g_tol, (ephi, eg)


def test_fmm_accuracy_amr_and_odd_dims(oracle_lib):
    """A refined octant (coarse leaves see the fine region through its
    restricted moments, fine leaves see coarse cells as uniform pieces) and a
    3 x 2 x 2 box inside a 4^3 root: same accuracy class as the uniform case,
    converging with R."""
    m = amr.amr_mesh(2, 2, 2, {(0, 1, 1, 0)})
    e2 = errors(oracle_lib, m.level, m.pos, m.dims, 1.0 / 16, 2)
    e3 = errors(oracle_lib, m.level, m.pos, m.dims, 1.0 / 16, 3)
    assert e2[0] < 3e-3 and e2[1] < 0.05 and e3[1] < e2[1]
    pos = grid_positions(3, 2, 2)
    e = errors(oracle_lib, np.zeros(12, np.int32), pos, (3, 2, 2), 1.0 / 16, 2)
    assert e[0] < 5e-3 and e[1] < 0.05


def test_fmm_single_root_leaf_is_the_direct_sum(oracle_lib):
    U = blob([0], [[0, 0, 0]], 1.0 / 8, centre=(0.5, 0.5, 0.5))
    f = oracle_lib.gravity_fmm(6, [0], [[0, 0, 0]], (1, 1, 1), 1.0 / 8, U, radius=2)
    d = oracle_lib.gravity_direct(6, [0], [[0, 0, 0]], (1, 1, 1), 1.0 / 8, U)
    assert np.allclose(f, d, rtol=1e-12, atol=1e-15)


def test_fmm_point_mass_far_field(oracle_lib):
    """One heavy cell in a 4^3 box of near-vacuum: the field far from it is
    the point mass's, g = -G m r / r^3, to the FMM's accuracy (here the
    first-order local expansion carried down two depths: ~0.8 %)."""
    pos = grid_positions(4, 4, 4)
    dx0 = 1.0 / 32
    U = np.zeros((64, 6, 512))
    U[:, 0] = 1e-12
    U[0, 0, 0] = 1.0 / dx0 ** 3  # unit mass at cell (0, 0, 0)
    f = oracle_lib.gravity_fmm(6, np.zeros(64, np.int32), pos, (4, 4, 4), dx0, U, radius=2)
    src = np.full(3, 0.5 * dx0)
    k, i = 63, 511  # the opposite corner cell
    x = (pos[k] * 8 + np.array([i & 7, (i >> 3) & 7, i >> 6]) + 0.5) * dx0
    r = x - src
    g = -r / np.linalg.norm(r) ** 3
    assert np.allclose(f[k, 1:, i], g, rtol=1.5e-2)
    assert abs(f[k, 0, i] + 1 / np.linalg.norm(r)) < 2e-3 / np.linalg.norm(r)


def test_fmm_rejects_malformed_trees(oracle_lib):
    U = np.zeros((2, 6, 512))
    with pytest.raises(ValueError):  # a leaf and its own child
        oracle_lib.gravity_fmm(6, [0, 1], [[0, 0, 0], [0, 0, 0]], (1, 1, 1), 1.0, U)
    with pytest.raises(ValueError):  # outside the domain
        oracle_lib.gravity_fmm(6, [0, 0], [[0, 0, 0], [2, 0, 0]], (2, 1, 1), 1.0, U)


def _leaves_of(level, pos):
    keys = {(int(l), *map(int, p)) for l, p in zip(level, pos)}
    refined = np.array([any((l + 1, 2 * p[0] + (c & 1), 2 * p[1] + ((c >> 1) & 1), 2 * p[2] + (c >> 2)) in keys
                            for c in range(8)) for l, p in zip(level, pos)])
    return refined


def test_gravity_tree_is_the_reference_octree(hydro, golden):
    """From the leaves of the reference's build_mesh octrees (golden, 2-4
    levels) the product's tree (ts_hydro_gravity_tree) rebuilds exactly the
    reference's grids, and names every node's gravity kernel as the reference's
    gravity_kernel_name does (workload.cpp:365-372; golden gravity_kind)."""
    vec, _ = golden
    for m in vec["build_mesh"]:
        lev, pos, kind = np.array(m["level"]), np.array(m["pos"]), np.array(m["gravity_kind"])
        refined = _leaves_of(lev, pos)
        t = hydro.gravity_tree(lev[~refined], pos[~refined], (1, 1, 1))
        mine = {(int(l), *map(int, p)): int(k) for l, p, k in zip(t["level"], t["pos"], t["kind"])}
        ref = {(int(l), *map(int, p)): int(k) for l, p, k in zip(lev, pos, kind)}
        assert mine == ref, m["levels"]
        leaf_nodes = t["leaf"] >= 0
        assert sorted(t["leaf"][leaf_nodes]) == list(range(int((~refined).sum())))


def test_gravity_tree_uniform_and_refusals(hydro):
    m = hydro.uniform_mesh(4, 3, 2)
    t = hydro.gravity_tree(np.zeros(m.n, np.int32), m.pos, m.dims)
    # 24 leaves at level 0 under a 4^3 root two virtual levels up: 1 + 4 + 24 nodes
    assert len(t["level"]) == 29 and sorted(set(t["level"])) == [-2, -1, 0]
    assert [hydro.GRAVITY_KINDS[k] for k in t["kind"][:1]] == ["multipole_root_kernel"]
    assert set(t["kind"][t["leaf"] >= 0]) == {3}
    with pytest.raises(ValueError):
        hydro.gravity_tree([0, 0], [[0, 0, 0], [0, 0, 0]], (1, 1, 1))


def test_self_gravity_cold_sphere_starts_homologous_collapse(oracle_lib):
    """A cold uniform sphere at rest: after one hydro + self-gravity step
    (oracle loop, the contract the GPU is held to bitwise) the momentum inside
    is the kick of g = -(4 pi / 3) G rho0 r: radial, linear in r."""
    nbr, pos, _ = oracle_lib.uniform_mesh(4, 4, 4)
    dx0 = 1.0 / 32
    i = np.arange(512)
    loc = np.stack([i & 7, (i >> 3) & 7, i >> 6]).astype(float)
    U = np.zeros((64, 6, 512))
    rho0, a = 1.0, 0.3
    for k in range(64):
        xc = (pos[k][:, None] * 8 + loc + 0.5) * dx0 - 0.5
        r = np.sqrt((xc ** 2).sum(0))
        U[k, 0] = np.where(r < a, rho0, 1e-3)
        U[k, 4] = 1e-6  # cold
    p = oracle_lib.params(nf=6, dx=dx0)
    U1, dts = oracle_lib.run_self_gravity(p, nbr, U, 1, np.zeros(64, np.int32),
                                          pos, (4, 4, 4), dx0, radius=2, G=1.0)
    dt = dts[0]
    want = -(4 * np.pi / 3) * rho0
    ratios = []
    for k in range(64):
        xc = (pos[k][:, None] * 8 + loc + 0.5) * dx0 - 0.5
        r = np.sqrt((xc ** 2).sum(0))
        inside = (r > 0.05) & (r < 0.5 * a)
        vr = (U1[k, 1:4] * xc).sum(0) / r / U1[k, 0]
        ratios.extend((vr[inside] / (r[inside] * dt)).tolist())
    ratios = np.array(ratios)
    assert len(ratios) > 100
    assert np.abs(ratios / want - 1).max() < 0.05, (ratios.min() / want, ratios.max() / want)
