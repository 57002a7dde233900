"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes front end of ``oracle/liboracle.so`` (the plain-C restatement in
``hydro_oracle.c``) and, when it was built, of ``oracle/_ref`` (the reference's
own core compiled from /root/reference).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may import this
package, and only as the checker / CPU baseline.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libtaskscope_ref.so")

N = 8
NC = 512

_lib = None
_ref = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_f64p = ctypes.POINTER(ctypes.c_double)


class Params(ctypes.Structure):
    _fields_ = [
        ("nf", ctypes.c_int32),
        ("recon", ctypes.c_int32),
        ("gamma", ctypes.c_double),
        ("cfl", ctypes.c_double),
        ("dx", ctypes.c_double),
        ("p_floor", ctypes.c_double),
    ]


def build(force: bool = False) -> None:
    srcs = [os.path.join(HERE, f) for f in ("hydro_oracle.c", "fmm_oracle.c", "hydro_oracle.h")]
    stale = os.path.exists(LIB_PATH) and all(os.path.exists(f) for f in srcs) and max(
        os.path.getmtime(f) for f in srcs) > os.path.getmtime(LIB_PATH)
    if force or stale or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)


def build_ref() -> bool:
    """Compile the reference core into oracle/_ref (only where /root/reference exists)."""
    if not os.path.isdir("/root/reference/proj/core/src"):
        return os.path.exists(REF_PATH)
    subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)
    return True


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        L.orc_mix64.restype = ctypes.c_uint64
        L.orc_mix64.argtypes = [ctypes.c_uint64]
        L.orc_mix64_2.restype = ctypes.c_uint64
        L.orc_mix64_2.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.orc_cell_value.restype = ctypes.c_double
        L.orc_cell_value.argtypes = [ctypes.c_uint64] * 3
        L.orc_face_cell_index.restype = ctypes.c_uint64
        L.orc_face_cell_index.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64]
        L.orc_morton3.restype = ctypes.c_uint64
        L.orc_morton3.argtypes = [ctypes.c_uint32] * 3
        L.orc_uniform_mesh.restype = ctypes.c_int
        L.orc_uniform_mesh.argtypes = [ctypes.c_int] * 7 + [_i64p, _i32p, _i32p]
        L.orc_exchange_faces.argtypes = [ctypes.c_int, ctypes.c_int64, _i64p, _f64p, _f64p]
        L.orc_fill_halo.argtypes = [ctypes.c_int, ctypes.c_int64, _i64p, _f64p, ctypes.c_int, _f64p]
        L.orc_max_signal_speed.restype = ctypes.c_double
        L.orc_max_signal_speed.argtypes = [ctypes.POINTER(Params), ctypes.c_int64, ctypes.c_int64, _f64p]
        L.orc_stage.argtypes = [ctypes.POINTER(Params), ctypes.c_int64, _i64p, _f64p, _f64p, _f64p,
                                ctypes.c_int, ctypes.c_double, ctypes.c_int64, ctypes.c_int64]
        L.orc_run.restype = ctypes.c_int
        L.orc_run.argtypes = [ctypes.POINTER(Params), ctypes.c_int64, _i64p, _f64p, ctypes.c_int,
                              _f64p, ctypes.c_int]
        L.orc_field_sums.argtypes = [ctypes.c_int, ctypes.c_int64, _f64p, _f64p]
        L.orc_ic_sod.argtypes = [ctypes.POINTER(Params), ctypes.c_int64, _i32p, ctypes.c_int, _f64p]
        L.orc_ic_sedov.argtypes = [ctypes.POINTER(Params), ctypes.c_int64, _i32p, ctypes.c_int,
                                   ctypes.c_int, ctypes.c_int, _f64p]
        L.orc_ic_random.argtypes = [ctypes.POINTER(Params), ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_uint64, _f64p]
        L.orc_ic_polytrope.argtypes = [ctypes.POINTER(Params), ctypes.c_int64, _i32p, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, _f64p]
        L.orc_ic_binary.restype = ctypes.c_int
        L.orc_ic_binary.argtypes = [ctypes.POINTER(Params), ctypes.c_int64, _i32p, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, _f64p]
        L.orc_p2p_stencil.restype = ctypes.c_int
        L.orc_p2p_stencil.argtypes = [ctypes.c_int, _i32p, _f64p, ctypes.c_int]
        L.orc_gravity_p2p.argtypes = [ctypes.POINTER(Params), ctypes.c_int64, _i64p, _f64p, ctypes.c_int,
                                      ctypes.c_double, _f64p]
        L.orc_fmm_table.restype = ctypes.c_int
        L.orc_fmm_table.argtypes = [ctypes.c_int, ctypes.c_int, _i32p, _i32p, ctypes.c_int]
        for fn in (L.orc_gravity_fmm, L.orc_gravity_direct):
            fn.restype = ctypes.c_int
        L.orc_gravity_fmm.argtypes = [ctypes.c_int, ctypes.c_int64, _i32p, _i32p, _i32p, ctypes.c_double, _f64p,
                                      ctypes.c_int, ctypes.c_double, _f64p]
        L.orc_gravity_direct.argtypes = [ctypes.c_int, ctypes.c_int64, _i32p, _i32p, _i32p, ctypes.c_double, _f64p,
                                         ctypes.c_double, _f64p]
        L.orc_gravity_kick.argtypes = [ctypes.c_int, ctypes.c_int64, _f64p, _f64p, ctypes.c_double]
        L.orc_amr_fill.argtypes = [ctypes.c_int, ctypes.c_int64, _i32p, _f64p]
        L.orc_amr_reflux.argtypes = [ctypes.POINTER(Params), _i64p, _i32p, ctypes.c_int, ctypes.c_int64, _i32p,
                                     _f64p, _f64p, ctypes.c_int, ctypes.c_double]
        L.orc_run_amr.restype = ctypes.c_int
        L.orc_run_amr.argtypes = [ctypes.POINTER(Params), ctypes.c_int64, _i64p, _i32p, _i64p, ctypes.c_int,
                                  ctypes.c_int64, _i32p, ctypes.c_int64, _i32p, _f64p, ctypes.c_int, _f64p]
        _lib = L
    return _lib


def ref():
    """The compiled reference (oracle/_ref) or None when it was never built."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_PATH):
            return None
        R = ctypes.CDLL(REF_PATH)
        R.ref_mix64.restype = ctypes.c_uint64
        R.ref_mix64.argtypes = [ctypes.c_uint64]
        R.ref_mix64_2.restype = ctypes.c_uint64
        R.ref_mix64_2.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        R.ref_cell_value.restype = ctypes.c_double
        R.ref_cell_value.argtypes = [ctypes.c_uint64] * 3
        R.ref_face_cell_index.restype = ctypes.c_uint64
        R.ref_face_cell_index.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64]
        R.ref_gravity_kinds.restype = ctypes.c_int64
        R.ref_gravity_kinds.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, _i32p, ctypes.c_int64]
        R.ref_build_mesh.restype = ctypes.c_int64
        R.ref_build_mesh.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, _i32p, _i32p, _i32p,
                                     _i64p, ctypes.c_int64]
        R.ref_exchange_ghosts.restype = ctypes.c_int
        R.ref_exchange_ghosts.argtypes = [ctypes.c_int64, _i64p, _i32p, _i32p, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_uint64, _f64p, _u64p]
        R.ref_fill_cells.argtypes = [ctypes.c_int64, ctypes.c_uint64, _f64p]
        _ref = R
    return _ref


def _p(a, t):
    return a.ctypes.data_as(t)


def params(nf=6, recon=0, gamma=1.4, cfl=0.4, dx=1.0 / 32, p_floor=1e-12) -> Params:
    return Params(nf, recon, gamma, cfl, dx, p_floor)


def uniform_mesh(nx, ny, nz, periodic=(False, False, False), world=1):
    n = nx * ny * nz
    nbr = np.zeros((n, 6), np.int64)
    pos = np.zeros((n, 3), np.int32)
    owner = np.zeros(n, np.int32)
    rc = lib().orc_uniform_mesh(nx, ny, nz, int(periodic[0]), int(periodic[1]), int(periodic[2]), world,
                                _p(nbr, _i64p), _p(pos, _i32p), _p(owner, _i32p))
    if rc != 0:
        raise ValueError("bad mesh dimensions")
    return nbr, pos, owner


def ic_sod(p: Params, pos, axis=0):
    U = np.zeros((len(pos), p.nf, NC), np.float64)
    lib().orc_ic_sod(ctypes.byref(p), len(pos), _p(np.ascontiguousarray(pos), _i32p), axis, _p(U, _f64p))
    return U


def ic_sedov(p: Params, pos, dims):
    U = np.zeros((len(pos), p.nf, NC), np.float64)
    lib().orc_ic_sedov(ctypes.byref(p), len(pos), _p(np.ascontiguousarray(pos), _i32p), dims[0], dims[1],
                       dims[2], _p(U, _f64p))
    return U


def ic_random(p: Params, g_begin, g_end, seed=2210):
    U = np.zeros((g_end - g_begin, p.nf, NC), np.float64)
    lib().orc_ic_random(ctypes.byref(p), g_begin, g_end, seed, _p(U, _f64p))
    return U


def ic_polytrope(p: Params, pos, dims):
    U = np.zeros((len(pos), p.nf, NC), np.float64)
    lib().orc_ic_polytrope(ctypes.byref(p), len(pos), _p(np.ascontiguousarray(pos), _i32p), dims[0], dims[1],
                           dims[2], _p(U, _f64p))
    return U


def ic_binary(p: Params, pos, dims):
    U = np.zeros((len(pos), p.nf, NC), np.float64)
    if lib().orc_ic_binary(ctypes.byref(p), len(pos), _p(np.ascontiguousarray(pos), _i32p), dims[0], dims[1],
                           dims[2], _p(U, _f64p)) != 0:
        raise MemoryError("oracle binary initial model")
    return U


def p2p_stencil(radius):
    """The gravity P2P stencil of radius R: offsets [n][3] and coefficients
    [n][4] = (1/|d|, d/|d|^3) in the summation order (hydro_oracle.h)."""
    off = np.zeros((1024, 3), np.int32)
    coef = np.zeros((1024, 4), np.float64)
    n = lib().orc_p2p_stencil(radius, _p(off, _i32p), _p(coef, _f64p), 1024)
    if n < 0:
        raise ValueError("radius outside 1..6")
    return off[:n], coef[:n]


def gravity_p2p(p: Params, nbr, U, radius=4, G=1.0):
    """Near-field monopole potential and acceleration: [n][4][512] = (phi, gx, gy, gz)."""
    nbr = np.ascontiguousarray(nbr, np.int64)
    U = np.ascontiguousarray(U, np.float64)
    out = np.zeros((U.shape[0], 4, NC), np.float64)
    lib().orc_gravity_p2p(ctypes.byref(p), U.shape[0], _p(nbr, _i64p), _p(U, _f64p), radius, G, _p(out, _f64p))
    return out


def fmm_table(radius, root=False):
    """FMM interaction table (octant-0 orientation): offsets [n][3] and near flags [n]."""
    u = np.zeros((4096, 3), np.int32)
    near = np.zeros(4096, np.int32)
    n = lib().orc_fmm_table(radius, int(root), _p(u, _i32p), _p(near, _i32p), 4096)
    if n < 0:
        raise ValueError("radius outside 1..3")
    return u[:n], near[:n].astype(bool)


def _leaves(level, pos, dims):
    level = np.ascontiguousarray(level, np.int32)
    pos = np.ascontiguousarray(np.asarray(pos).reshape(-1, 3), np.int32)
    dims = np.ascontiguousarray(dims, np.int32)
    return level, pos, dims


def gravity_fmm(nf, level, pos, dims, dx0, U, radius=2, G=1.0):
    """Whole gravity solve (FMM, fmm_oracle.c): [n][4][512] = (phi, gx, gy, gz) per leaf."""
    level, pos, dims = _leaves(level, pos, dims)
    U = np.ascontiguousarray(U, np.float64)
    out = np.zeros((len(level), 4, NC), np.float64)
    if lib().orc_gravity_fmm(nf, len(level), _p(level, _i32p), _p(pos, _i32p), _p(dims, _i32p), dx0,
                             _p(U, _f64p), radius, G, _p(out, _f64p)) != 0:
        raise ValueError("malformed gravity tree (overlapping leaves or positions outside the domain)")
    return out


def gravity_kick(U, grav, dt):
    """Gravity source over dt (orc_gravity_kick) on a copy of U."""
    U = np.array(U, np.float64, copy=True, order="C")
    grav = np.ascontiguousarray(grav, np.float64)
    assert grav.shape[0] >= U.shape[0]
    lib().orc_gravity_kick(U.shape[1], U.shape[0], _p(U, _f64p), _p(grav, _f64p), dt)
    return U


def run_self_gravity(p: Params, nbr, U, nsteps, level, pos, dims, dx0, radius=2, G=1.0, mesh=None):
    """Hydro with self-gravity, the order ts_hydro_step_gravity follows: per
    step one SSP-RK3 hydro step (dt from the state), the FMM on the result, the
    kick over that dt.  mesh: an AmrMesh (then nbr is ignored and U holds the
    leaves).  Returns (U, dts)."""
    U = np.array(U, np.float64, copy=True, order="C")
    dts = []
    for _ in range(nsteps):
        if mesh is None:
            U, dt = run(p, nbr, U, 1)
        else:
            full = np.zeros((mesh.n_total,) + U.shape[1:])
            full[:mesh.n_leaves] = U
            full, dt = run_amr(p, mesh, full, 1)
            U = full[:mesh.n_leaves].copy()
        g = gravity_fmm(U.shape[1], level, pos, dims, dx0, U, radius=radius, G=G)
        U = gravity_kick(U, g, dt[0])
        dts.append(dt[0])
    return U, np.array(dts)


def gravity_direct(nf, level, pos, dims, dx0, U, G=1.0):
    """Brute-force pair sum over every leaf cell (the FMM's accuracy yardstick)."""
    level, pos, dims = _leaves(level, pos, dims)
    U = np.ascontiguousarray(U, np.float64)
    out = np.zeros((len(level), 4, NC), np.float64)
    lib().orc_gravity_direct(nf, len(level), _p(level, _i32p), _p(pos, _i32p), _p(dims, _i32p), dx0,
                             _p(U, _f64p), G, _p(out, _f64p))
    return out


def max_signal_speed(p: Params, U):
    U = np.ascontiguousarray(U)
    return lib().orc_max_signal_speed(ctypes.byref(p), 0, U.shape[0], _p(U, _f64p))


def stage(p: Params, nbr, Uprev, Un, stage_no, dtdx, g_begin=0, g_end=None):
    nbr = np.ascontiguousarray(nbr, np.int64)
    Uprev = np.ascontiguousarray(Uprev)
    Un = np.ascontiguousarray(Un)
    out = np.zeros_like(Uprev)
    if g_end is None:
        g_end = Uprev.shape[0]
    lib().orc_stage(ctypes.byref(p), Uprev.shape[0], _p(nbr, _i64p), _p(Uprev, _f64p), _p(Un, _f64p),
                    _p(out, _f64p), stage_no, dtdx, g_begin, g_end)
    return out


def run(p: Params, nbr, U, nsteps, nthreads=1):
    """nsteps SSP-RK3 steps; returns (U_new, dt_history)."""
    nbr = np.ascontiguousarray(nbr, np.int64)
    U = np.array(U, np.float64, copy=True, order="C")
    dts = np.zeros(max(nsteps, 1), np.float64)
    rc = lib().orc_run(ctypes.byref(p), U.shape[0], _p(nbr, _i64p), _p(U, _f64p), nsteps, _p(dts, _f64p),
                       nthreads)
    if rc != 0:
        raise MemoryError("oracle run failed")
    return U, dts[:nsteps]


def field_sums(U):
    U = np.ascontiguousarray(U)
    s = np.zeros(U.shape[1], np.float64)
    lib().orc_field_sums(U.shape[1], U.shape[0], _p(U, _f64p), _p(s, _f64p))
    return s


def exchange_faces(nbr, U):
    U = np.ascontiguousarray(U)
    ghost = np.zeros((U.shape[0], 6, N * N), np.float64)
    lib().orc_exchange_faces(U.shape[1], U.shape[0], _p(np.ascontiguousarray(nbr, np.int64), _i64p),
                             _p(U, _f64p), _p(ghost, _f64p))
    return ghost


def fill_halo(nbr, U, h=3):
    U = np.ascontiguousarray(U)
    pe = N + 2 * h
    tiles = np.zeros((U.shape[0], U.shape[1], pe, pe, pe), np.float64)
    lib().orc_fill_halo(U.shape[1], U.shape[0], _p(np.ascontiguousarray(nbr, np.int64), _i64p),
                        _p(U, _f64p), h, _p(tiles, _f64p))
    return tiles


def to_global(U, pos, dims, field=0):
    """Assemble field `field` of a [g][nf][512] state into a [z][y][x] array."""
    nx, ny, nz = dims
    out = np.zeros((nz * N, ny * N, nx * N), np.float64)
    for g in range(U.shape[0]):
        x, y, z = pos[g]
        out[z * N:(z + 1) * N, y * N:(y + 1) * N, x * N:(x + 1) * N] = U[g, field].reshape(N, N, N)
    return out


def amr_fill(nf, mesh, U):
    """Proxy fill (prolongation / restriction) in place on U [n_total, nf, 512]."""
    px = np.ascontiguousarray(mesh.proxies, np.int32)
    lib().orc_amr_fill(nf, len(px), _p(px, _i32p), _p(U, _f64p))
    return U


def run_amr(p: Params, mesh, U, nsteps):
    """nsteps SSP-RK3 steps on an AMR mesh (paper_2210_06437_b200.amr.AmrMesh);
    U is [n_total, nf, 512] (proxy slots may hold anything).  Returns (U, dts)."""
    U = np.array(U, np.float64, copy=True, order="C")
    assert U.shape[0] == mesh.n_total
    nbr = np.zeros((mesh.n_total, 6), np.int64) - 1
    nbr[:mesh.n_leaves] = mesh.nbr
    lev = np.ascontiguousarray(mesh.level, np.int32)
    lf = np.ascontiguousarray(mesh.level_first, np.int64)
    px = np.ascontiguousarray(mesh.proxies, np.int32)
    rf = np.ascontiguousarray(mesh.reflux, np.int32)
    dts = np.zeros(max(nsteps, 1), np.float64)
    rc = lib().orc_run_amr(ctypes.byref(p), mesh.n_total, _p(nbr, _i64p), _p(lev, _i32p), _p(lf, _i64p),
                           mesh.max_level, len(px), _p(px, _i32p), len(rf), _p(rf, _i32p), _p(U, _f64p), nsteps,
                           _p(dts, _f64p))
    if rc != 0:
        raise MemoryError("oracle AMR run failed")
    return U, dts[:nsteps]


def amr_reflux(p: Params, mesh, Uprev, Uout, stage_no, dt):
    """orc_amr_reflux in place on Uout (both [n_total, nf, 512])."""
    nbr = np.zeros((mesh.n_total, 6), np.int64) - 1
    nbr[:mesh.n_leaves] = mesh.nbr
    lev = np.ascontiguousarray(mesh.level, np.int32)
    rf = np.ascontiguousarray(mesh.reflux, np.int32)
    Uprev = np.ascontiguousarray(Uprev)
    lib().orc_amr_reflux(ctypes.byref(p), _p(nbr, _i64p), _p(lev, _i32p), mesh.max_level, len(rf), _p(rf, _i32p),
                         _p(Uprev, _f64p), _p(Uout, _f64p), stage_no, dt)
    return Uout


def amr_stage(p: Params, mesh, Uprev, Un, stage_no, dt, reflux=True):
    """One AMR stage as orc_run_amr does it: fill proxies of Uprev (in place),
    per-level orc_stage, then the flux correction."""
    amr_fill(p.nf, mesh, Uprev)
    nbr = np.zeros((mesh.n_total, 6), np.int64) - 1
    nbr[:mesh.n_leaves] = mesh.nbr
    out = np.zeros_like(Uprev)
    for L in range(mesh.max_level + 1):
        f0, f1 = int(mesh.level_first[L]), int(mesh.level_first[L + 1])
        part = stage(p, nbr, Uprev, Un, stage_no, dt / np.ldexp(p.dx, mesh.max_level - L), f0, f1)
        out[f0:f1] = part[f0:f1]
    if reflux:
        amr_reflux(p, mesh, Uprev, out, stage_no, dt)
    return out
