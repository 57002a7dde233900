"""Coarse-fine AMR: mesh builder, the
oracle's prolongation / restriction / reflux, and the C-ABI validation of
ts_hydro_set_amr_mesh on a host-only context.  CPU only; the GPU parity of the
same runs is in test_gpu_amr.py."""
import numpy as np
import pytest

from paper_2210_06437_b200 import amr

DX = 1.0 / 64

# a 2x2x2 block of level-0 positions refined in the middle of a 4^3 box
CENTRE_BLOCK = {(0, x, y, z) for x in (1, 2) for y in (1, 2) for z in (1, 2)}
# an L-shaped refined region off-centre: coarse leaves see fine ones on 1-3 faces
L_SHAPE = {(0, 1, 1, 1), (0, 2, 1, 1), (0, 1, 2, 1), (0, 1, 1, 2), (0, 2, 2, 2)}


def totals(mesh, U, nf):
    vol = mesh.cell_volumes(DX)
    return np.array([(U[:mesh.n_leaves, f].sum(axis=1) * vol).sum() for f in range(nf)])


def test_builder_covers_the_domain_once():
    for refine in (CENTRE_BLOCK, L_SHAPE, set()):
        m = amr.amr_mesh(4, 4, 4, refine)
        ext = 4 * 8 * DX * 2 ** m.max_level
        assert np.isclose(m.cell_volumes(DX).sum() * 512, ext ** 3, rtol=1e-15, atol=0)
        assert (np.diff(m.level) >= 0).all()
        assert m.level_first[-1] == m.n_leaves
        # same-level leaf links are symmetric; proxies only across levels
        for i in range(m.n_leaves):
            for f in range(6):
                nb = m.nbr[i, f]
                if 0 <= nb < m.n_leaves:
                    assert m.nbr[nb, f ^ 1] == i and m.level[nb] == m.level[i]


def test_builder_proxies_and_reflux_records():
    m = amr.amr_mesh(4, 4, 4, L_SHAPE)
    assert m.n_proxy > 0 and len(m.reflux) > 0
    kinds = m.proxies[:, 1]
    assert set(kinds.tolist()) == {0, 1}
    for r in m.proxies:
        dst, kind, octant, src = r[0], r[1], r[2], r[3:]
        assert m.n_leaves <= dst < m.n_total
        if kind == 0:
            assert m.level[src[0]] == 0 and 0 <= octant < 8
        else:
            assert (m.level[src] == 1).all()
            # children in octant order: positions 2q + o
            base = m.pos[src[0]]
            for o in range(8):
                assert tuple(m.pos[src[o]]) == (base[0] + (o & 1), base[1] + ((o >> 1) & 1), base[2] + (o >> 2))
    for rec in m.reflux:
        g, fine = rec[0], rec[1:].reshape(6, 4)
        assert m.level[g] == 0
        for f in range(6):
            if fine[f, 0] < 0:
                continue
            axis, side = f >> 1, f & 1
            for k in fine[f]:
                assert m.level[k] == 1
                # the fine leaf touches the coarse face
                lo = m.pos[g] * 2
                fp = m.pos[k]
                assert fp[axis] == (lo[axis] + 2 if side else lo[axis] - 1)


def test_unbalanced_mesh_is_rejected():
    with pytest.raises(ValueError, match="2:1"):
        amr.amr_mesh(4, 4, 4, lambda L, p: p == (1, 1, 1) or (L == 1 and p == (2, 2, 2)), max_level=2)


def test_unrefined_amr_run_is_the_uniform_run(oracle_lib):
    """No refinement: the AMR driver reduces to orc_run bitwise."""
    m = amr.amr_mesh(4, 4, 4, set())
    assert m.n_proxy == 0
    nbr, pos, _ = oracle_lib.uniform_mesh(4, 4, 4)
    assert (nbr == m.nbr).all() and (pos == m.pos).all()
    p = oracle_lib.params(nf=6, dx=DX * 2)
    U0 = amr.ic_blast(m, 6, DX * 2)
    Ua, da = oracle_lib.run_amr(p, m, U0, 3)
    Uu, du = oracle_lib.run(p, nbr, U0, 3)
    assert np.array_equal(Ua, Uu) and np.array_equal(da, du)


def test_fully_refined_amr_run_is_the_fine_uniform_run(oracle_lib):
    """Every level-0 position refined: a uniform level-1 mesh, bitwise."""
    m = amr.amr_mesh(2, 2, 2, lambda L, p: True)
    assert m.n_proxy == 0 and (m.level == 1).all()
    nbr, pos, _ = oracle_lib.uniform_mesh(4, 4, 4)
    p = oracle_lib.params(nf=6, dx=DX)
    U0 = amr.ic_blast(m, 6, DX, drift=(0.3, -0.2, 0.1))
    at = {tuple(q): i for i, q in enumerate(pos)}
    perm = np.array([at[tuple(q)] for q in m.pos])  # leaf -> uniform id
    Uu0 = np.empty_like(U0)
    Uu0[perm] = U0
    Ua, da = oracle_lib.run_amr(p, m, U0, 2)
    Uu, du = oracle_lib.run(p, nbr, Uu0, 2)
    assert np.array_equal(Ua, Uu[perm]) and np.array_equal(da, du)


# bump centred on a coarse-fine face, >= 0.375 (12 coarse cells) from the
# outflow boundary: closer, the boundary itself leaks ~1e-12 in 5 steps on a
# uniform mesh too
CENTRE_BLOCK6 = {(0, x, y, z) for x in (2, 3) for y in (2, 3) for z in (2, 3)}
CF_CASES = [((6, 6, 6), CENTRE_BLOCK6, (1.0, 0.75, 0.75)), ((4, 4, 4), L_SHAPE, (0.625, 0.625, 0.5))]


@pytest.mark.parametrize("dims,refine,centre", CF_CASES, ids=["centre", "lshape"])
@pytest.mark.parametrize("recon", [0, 1])
def test_reflux_conserves_to_round_off(oracle_lib, dims, refine, centre, recon):
    m = amr.amr_mesh(*dims, refine)
    p = oracle_lib.params(nf=6, recon=recon, dx=DX)
    U0 = amr.ic_blast(m, 6, DX, width=0.04, centre=centre)
    # the bump sits on a coarse-fine face and its tail at the outflow
    # boundary is ~1e-17, so mass, momentum and energy only move between cells
    t0 = totals(m, U0, 6)
    U, _ = oracle_lib.run_amr(p, m, U0, 5)
    err = np.abs(totals(m, U, 6) - t0)[:5] / np.abs(t0).max()
    assert err.max() < 1e-14, err
    # without the flux correction the coarse-fine faces leak
    m0 = amr.AmrMesh(m.dims, m.max_level, m.level, m.pos, m.nbr, m.level_first, m.proxies, m.reflux[:0])
    U_nofix, _ = oracle_lib.run_amr(p, m0, U0, 5)
    leak = np.abs(totals(m, U_nofix, 6) - t0)[[0, 4]] / np.abs(t0).max()
    assert leak.min() > 1e-8, leak


# three levels: a refined 2^3 level-0 block with its central 2^3 level-1
# positions refined again (restrictions with further-refined far children)
def THREE_LEVELS(L, p):
    return (L == 0 and all(1 <= v <= 2 for v in p)) or (L == 1 and all(3 <= v <= 4 for v in p))


def test_three_level_mesh_conserves_and_keeps_free_stream(oracle_lib):
    m = amr.amr_mesh(4, 4, 4, THREE_LEVELS, max_level=2)
    assert m.max_level == 2 and list(np.diff(m.level_first)) == [56, 56, 64]
    dx = DX / 2
    vol = m.cell_volumes(dx)
    p = oracle_lib.params(nf=6, dx=dx)
    U0 = amr.ic_blast(m, 6, dx, width=0.05, centre=(0.5, 0.5, 0.5))
    t = lambda U: np.array([(U[:m.n_leaves, f].sum(axis=1) * vol).sum() for f in range(5)])  # noqa: E731
    U, _ = oracle_lib.run_amr(p, m, U0, 3)
    assert (np.abs(t(U) - t(U0)) / np.abs(t(U0)).max()).max() < 1e-14
    U0 = amr.ic_blast(m, 6, dx, amp=0.0, drift=(0.5, -0.25, 0.125))
    U, _ = oracle_lib.run_amr(p, m, U0, 2)
    for f in range(6):
        assert (U[:m.n_leaves, f] == U0[0, f, 0]).all(), f


def test_uniform_flow_stays_uniform_across_levels(oracle_lib):
    """Free-stream preservation: prolongation, restriction and reflux of a
    uniform state are exact, so every cell keeps its bits."""
    m = amr.amr_mesh(4, 4, 4, L_SHAPE)
    p = oracle_lib.params(nf=8, dx=DX)
    U0 = amr.ic_blast(m, 8, DX, amp=0.0, drift=(0.5, -0.25, 0.125))
    U0[:m.n_leaves, 6:] = 0.3
    U, _ = oracle_lib.run_amr(p, m, U0, 4)
    for f in range(8):
        assert (U[:m.n_leaves, f] == U0[0, f, 0]).all(), f


def test_fill_prolongs_and_restricts(oracle_lib):
    m = amr.amr_mesh(2, 2, 2, {(0, 0, 0, 0)})
    U = np.zeros((m.n_total, 6, 512))
    rng = np.random.default_rng(5)
    U[:m.n_leaves] = rng.random((m.n_leaves, 6, 512)) + 1
    oracle_lib.amr_fill(6, m, U)
    i = np.arange(512)
    x, y, z = i & 7, (i >> 3) & 7, i >> 6
    for r in m.proxies:
        dst, kind, octant, src = r[0], r[1], r[2], r[3:]
        if kind == 0:
            cc = ((octant >> 2 & 1) * 4 + z // 2) * 64 + ((octant >> 1 & 1) * 4 + y // 2) * 8 + (octant & 1) * 4 + x // 2
            assert np.array_equal(U[dst], U[src[0]][:, cc])
        else:
            o = (x >> 2) | ((y >> 2) << 1) | ((z >> 2) << 2)
            fine = U[src[o]]  # [512(cell), 6, 512] per proxy cell
            bx, by, bz = 2 * (x & 3), 2 * (y & 3), 2 * (z & 3)
            mean = sum(fine[np.arange(512), :, (bz + k) * 64 + (by + j) * 8 + bx + ii]
                       for k in (0, 1) for j in (0, 1) for ii in (0, 1)) / 8
            assert np.allclose(U[dst].T, mean, rtol=1e-15, atol=0)


def test_set_amr_mesh_validates(hydro):
    m = amr.amr_mesh(4, 4, 4, L_SHAPE)
    d = hydro.CudaDevice(hydro.HydroConfig(device_id=-1))
    d.set_amr_mesh(m)
    assert d.local_counts()[:2] == (m.n_leaves, m.n_proxy)

    def bad(**kw):
        f = dict(nbr=m.nbr, level=m.level, proxies=m.proxies, reflux=m.reflux)
        f.update(kw)
        return amr.AmrMesh(m.dims, m.max_level, f["level"], m.pos, f["nbr"], m.level_first, f["proxies"],
                           f["reflux"])

    lev = m.level.copy()
    lev[0] = 1
    with pytest.raises(ValueError, match="level-major"):
        d.set_amr_mesh(bad(level=lev))
    nbr = m.nbr.copy()
    nbr[0, 1] = m.n_total + 3
    with pytest.raises(ValueError, match="out of range"):
        d.set_amr_mesh(bad(nbr=nbr))
    px = m.proxies.copy()
    px[0, 1] = 7
    with pytest.raises(ValueError, match="kind"):
        d.set_amr_mesh(bad(proxies=px))
    px = m.proxies.copy()
    px[0, 3] = m.n_leaves + 1
    with pytest.raises(ValueError, match="not a leaf"):
        d.set_amr_mesh(bad(proxies=px))
    rf = m.reflux.copy()
    f = next(k for k in range(6) if rf[0, 1 + 4 * k] >= 0)
    rf[0, 1 + 4 * f] = rf[0, 0]
    with pytest.raises(ValueError, match="one level finer"):
        d.set_amr_mesh(bad(reflux=rf))


def test_reference_build_mesh_octrees_become_amr_leaf_meshes(golden):
    """The reference's own octrees (build_mesh output, golden vectors drawn
    from the compiled reference): the leaves are the nodes without children,
    every same-level link between two leaves is the reference's link
    (workload.cpp:306-314), and the 2:1 balance the TreeBuilder enforces
    (workload.cpp:234-248) is accepted."""
    vec, _ = golden
    for m in vec["build_mesh"]:
        lvl = np.asarray(m["level"])
        pos = np.asarray(m["pos"]).reshape(-1, 3)
        nbr = np.asarray(m["nbr"]).reshape(-1, 6)
        a = amr.from_reference_mesh(lvl, pos)
        parents = {(int(L) - 1, *(int(v) >> 1 for v in p)) for L, p in zip(lvl, pos) if L > 0}
        ref_leaf = {(int(L), *map(int, p)): i for i, (L, p) in enumerate(zip(lvl, pos))
                    if (int(L), *map(int, p)) not in parents}
        ours = {(int(L), *map(int, p)): i for i, (L, p) in enumerate(zip(a.level, a.pos))}
        assert set(ours) == set(ref_leaf)
        for key, i in ours.items():
            r = ref_leaf[key]
            for f in range(6):
                rn = int(nbr[r, f])
                rkey = (int(lvl[rn]), *map(int, pos[rn])) if rn >= 0 else None
                if rkey is not None and rkey in ref_leaf:
                    # a same-level leaf neighbour in the reference: the same leaf here
                    assert a.nbr[i, f] >= 0 and a.nbr[i, f] < a.n_leaves
                    assert (int(a.level[a.nbr[i, f]]), *map(int, a.pos[a.nbr[i, f]])) == rkey
                elif a.nbr[i, f] >= 0 and a.nbr[i, f] < a.n_leaves:
                    raise AssertionError(f"leaf {key} face {f}: a same-level leaf link the reference lacks")


def test_reference_octree_amr_oracle_conserves_and_keeps_free_stream(oracle_lib, golden):
    """The AMR oracle on the reference's levels-4 octree: a uniform drifting
    state stays uniform bit for bit across the coarse-fine faces."""
    vec, _ = golden
    m = max(vec["build_mesh"], key=lambda e: len(e["level"]))
    a = amr.from_reference_mesh(m["level"], m["pos"])
    dx = 1.0 / (8 << a.max_level)
    U = np.zeros((a.n_total, 6, 512))
    U[:, 0] = 1.0
    U[:, 1] = 0.3
    U[:, 4] = 2.0
    out, _ = oracle_lib.run_amr(oracle_lib.params(nf=6, dx=dx), a, U, 2)
    assert np.array_equal(out[:a.n_leaves], U[:a.n_leaves])


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_amr_plans_pair_up_across_ranks(hydro, golden, world):
    """Multi-rank AMR host plans (ts_hydro_set_amr_mesh_partitioned on
    host-only contexts): the reference's Morton deal over the leaves of its
    own levels-4 octree; every whole-sub-grid ghost a rank receives from a
    peer is exactly what that peer sends it, in the same order."""
    vec, _ = golden
    m = max(vec["build_mesh"], key=lambda e: len(e["level"]))
    a = amr.from_reference_mesh(m["level"], m["pos"])
    owner = amr.partition(a, world)
    assert np.bincount(owner).tolist() == [len(owner) // world + (1 if r < len(owner) % world else 0)
                                           for r in range(world)]
    plans = []
    for r in range(world):
        d = hydro.CudaDevice(hydro.HydroConfig(device_id=-1))
        d.set_amr_mesh(a, owner=owner, rank=r, world=world)
        n_owned, n_extra, _ = d.local_counts()
        assert n_owned == int((owner == r).sum())
        plans.append({q: d.halo_plan(q) for q in range(world) if q != r})
        d.close()
    for r in range(world):
        for q in range(world):
            if q == r:
                continue
            send_rq = plans[r][q][0]
            recv_qr = plans[q][r][1]
            assert np.array_equal(send_rq, recv_qr)
            assert (send_rq[:, 1] == 6).all()  # whole sub-grids
            assert (owner[send_rq[:, 0]] == r).all()
