"""Gravity slice: the near-field monopole P2P the
reference's p2p_kernel launches stand for (workload.cpp:365-372, 565-569;
PAPER.md:355).  CPU tests pin the oracle restatement (hydro_oracle.h) with
known answers; tests/test_gpu_gravity.py holds the GPU parity."""
import numpy as np
import pytest


def test_stencil_is_a_sphere_ordered_by_radius(oracle_lib):
    for R in range(1, 7):
        off, coef = oracle_lib.p2p_stencil(R)
        r2 = (off.astype(np.int64) ** 2).sum(axis=1)
        assert (r2 >= 1).all() and (r2 <= R * R).all()
        assert len(off) == sum(1 for x in range(-R, R + 1) for y in range(-R, R + 1) for z in range(-R, R + 1)
                               if 0 < x * x + y * y + z * z <= R * R)
        assert (np.diff(r2) >= 0).all()  # |d|^2 ascending: the stencil of R is a prefix of the larger ones
        big, bigc = oracle_lib.p2p_stencil(6)
        assert np.array_equal(big[:len(off)], off) and np.array_equal(bigc[:len(off)], coef)
        assert np.array_equal(coef[:, 0], 1.0 / np.sqrt(r2.astype(np.float64)))
    with pytest.raises(ValueError):
        oracle_lib.p2p_stencil(7)


def _mesh(oracle_lib, dims, periodic=(False, False, False)):
    nbr, pos, _ = oracle_lib.uniform_mesh(*dims, periodic=periodic)
    return nbr, pos


def _global(U, pos, dims):
    n = np.array(dims) * 8
    G = np.zeros((n[2], n[1], n[0]))
    for g, p in enumerate(pos):
        G[p[2] * 8:(p[2] + 1) * 8, p[1] * 8:(p[1] + 1) * 8, p[0] * 8:(p[0] + 1) * 8] = U[g].reshape(8, 8, 8)
    return G


def test_single_mass_gives_the_point_mass_field(oracle_lib):
    """One cell of density 1 (mass h^3): phi = -G m / r and g = -G m (x_i - x_j) / r^3
    at every cell within R, nothing beyond — across sub-grid faces, edges and corners."""
    dims = (2, 2, 2)
    nbr, pos = _mesh(oracle_lib, dims)
    h, G, R = 1.0 / 16, 2.5, 4
    U = np.zeros((8, 6, 512))
    src = (7, 8, 9)  # global cell (x, y, z): next to a sub-grid corner
    for g, p in enumerate(pos):
        loc = [src[d] - 8 * p[d] for d in range(3)]
        if all(0 <= v < 8 for v in loc):
            U[g, 0, (loc[2] * 8 + loc[1]) * 8 + loc[0]] = 1.0
    out = oracle_lib.gravity_p2p(oracle_lib.params(nf=6, dx=h), nbr, U, radius=R, G=G)
    phi = _global(out[:, 0], pos, dims)
    gx = _global(out[:, 1], pos, dims)
    for z in range(16):
        for y in range(16):
            for x in range(16):
                d = (src[0] - x, src[1] - y, src[2] - z)  # offset of the source seen from the target
                r2 = d[0] ** 2 + d[1] ** 2 + d[2] ** 2
                if r2 == 0 or r2 > R * R:
                    assert phi[z, y, x] == 0.0 and gx[z, y, x] == 0.0
                    continue
                c0 = 1.0 / np.sqrt(float(r2))
                assert phi[z, y, x] == (-G * (h * h)) * c0
                assert gx[z, y, x] == (G * h) * (d[0] * (c0 / r2))  # pulls towards the source


def test_newtons_third_law(oracle_lib):
    """m_A g_A = -m_B g_B to rounding (c(-d) = -c(d) exactly; the products round once each)."""
    dims = (2, 1, 1)
    nbr, pos = _mesh(oracle_lib, dims)
    U = np.zeros((2, 6, 512))
    U[0, 0, (3 * 8 + 4) * 8 + 6] = 1.7    # cell (6, 4, 3) of sub-grid 0
    U[1, 0, (5 * 8 + 2) * 8 + 1] = 0.3    # cell (9, 2, 5) globally
    out = oracle_lib.gravity_p2p(oracle_lib.params(nf=6, dx=0.1), nbr, U, radius=5, G=1.0)
    ia, ib = (3 * 8 + 4) * 8 + 6, (5 * 8 + 2) * 8 + 1
    for k in (1, 2, 3):
        a, b = 1.7 * out[0, k, ia], -(0.3 * out[1, k, ib])
        assert a != 0.0 and abs(a - b) <= 4e-16 * abs(a)


@pytest.mark.parametrize("periodic", [(False, False, False), (True, True, True)])
def test_matches_a_brute_force_sum_on_the_global_grid(oracle_lib, periodic):
    dims = (2, 2, 2)
    nbr, pos = _mesh(oracle_lib, dims, periodic)
    rng = np.random.default_rng(7)
    U = np.zeros((8, 6, 512))
    U[:, 0] = rng.random((8, 512)) + 0.1
    h, G, R = 1.0 / 16, 1.3, 4
    out = oracle_lib.gravity_p2p(oracle_lib.params(nf=6, dx=h), nbr, U, radius=R, G=G)
    rho = _global(U[:, 0], pos, dims)
    off, _ = oracle_lib.p2p_stencil(R)
    n = 16
    phi = np.zeros_like(rho)
    g = np.zeros((3,) + rho.shape)
    zz, yy, xx = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    for dx, dy, dz in off:
        X, Y, Z = xx + dx, yy + dy, zz + dz
        if periodic[0]:
            X, Y, Z = X % n, Y % n, Z % n
            valid = np.ones_like(X, bool)
        else:
            valid = (X >= 0) & (X < n) & (Y >= 0) & (Y < n) & (Z >= 0) & (Z < n)
        src = np.where(valid, rho[np.clip(Z, 0, n - 1), np.clip(Y, 0, n - 1), np.clip(X, 0, n - 1)], 0.0)
        r = np.sqrt(dx * dx + dy * dy + dz * dz)
        phi += -G * h * h * src / r
        for k, d in enumerate((dx, dy, dz)):
            g[k] += G * h * src * d / r ** 3
    assert np.allclose(_global(out[:, 0], pos, dims), phi, rtol=1e-12, atol=0)
    for k in range(3):
        assert np.allclose(_global(out[:, 1 + k], pos, dims), g[k], rtol=1e-11, atol=1e-14)
