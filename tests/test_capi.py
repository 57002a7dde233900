"""C-ABI library checks that need no GPU: symbols, host-side mesh / IC /
halo-plan logic (against the oracle), config parsing and error behaviour."""
import os
import re

import numpy as np
import pytest

from tests.conftest import ROOT


def _declared_functions():
    with open(os.path.join(ROOT, "include", "ts_hydro.h")) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ts_hydro_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol(hydro):
    import ctypes
    L = ctypes.CDLL(hydro.LIB_PATH)
    names = _declared_functions()
    assert len(names) >= 35
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    # and the Python binding covers all of them
    assert set(names) <= set(hydro._SIGNATURES), set(names) - set(hydro._SIGNATURES)


def test_abi_version_and_strerror(hydro):
    L = hydro.lib()
    assert L.ts_hydro_abi_version() == 1
    assert L.ts_hydro_strerror(2) == b"device is shut down"
    assert L.ts_hydro_clock_ns() > 0


def test_kernel_image_is_sm100a(hydro):
    """The shipped library carries sm_100a SASS (no PTX-only / other-arch fallback)."""
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump")
    if tool is None:
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", hydro.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "stage_kernel" in subprocess.run([tool, "--list-text", hydro.LIB_PATH], capture_output=True,
                                            text=True).stdout or "sm_100a" in out


@pytest.mark.parametrize("dims,periodic,world", [((4, 4, 4), "", 1), ((3, 2, 5), "xz", 3), ((8, 1, 1), "x", 2),
                                                 ((16, 16, 16), "", 4)])
def test_uniform_mesh_matches_oracle(hydro, oracle_lib, dims, periodic, world):
    m = hydro.uniform_mesh(*dims, periodic=periodic, world=world)
    nbr, pos, owner = oracle_lib.uniform_mesh(*dims, tuple(ax in periodic for ax in "xyz"), world)
    assert np.array_equal(m.neighbor_ids, nbr)
    assert np.array_equal(m.pos, pos)
    assert np.array_equal(m.owner, owner)


@pytest.mark.parametrize("problem", ["sod", "sedov", "random", "polytrope", "binary"])
def test_ic_fill_matches_oracle_bitwise(hydro, oracle_lib, problem):
    species = {"random": 2, "polytrope": 5, "binary": 5}.get(problem, 0)
    cfg = hydro.HydroConfig(dx=1.0 / 32, n_species=species)
    m = hydro.uniform_mesh(4, 4, 4) if problem != "binary" else hydro.uniform_mesh(8, 4, 4)
    U = hydro.ic_fill(cfg, problem, m, np.arange(m.n), seed=2210)
    p = oracle_lib.params(nf=cfg.nf, dx=cfg.dx)
    if problem == "sod":
        want = oracle_lib.ic_sod(p, m.pos, 0)
    elif problem == "sedov":
        want = oracle_lib.ic_sedov(p, m.pos, (4, 4, 4))
    elif problem == "polytrope":
        want = oracle_lib.ic_polytrope(p, m.pos, (4, 4, 4))
    elif problem == "binary":
        want = oracle_lib.ic_binary(p, m.pos, (8, 4, 4))
    else:
        want = oracle_lib.ic_random(p, 0, m.n, 2210)
    assert np.array_equal(U, want)


def test_polytrope_and_binary_ics_are_physical(hydro):
    m = hydro.uniform_mesh(4, 4, 4)
    for prob, species in (("polytrope", 5), ("binary", 5)):
        cfg = hydro.HydroConfig(dx=1.0 / 32, n_species=species)
        U = hydro.ic_fill(cfg, prob, m, np.arange(m.n))
        assert np.isfinite(U).all()
        assert (U[:, 0] > 0).all()                       # density floor
        rho, E = U[:, 0], U[:, 4]
        ke = 0.5 * (U[:, 1] ** 2 + U[:, 2] ** 2 + U[:, 3] ** 2) / rho
        assert (E - ke > 0).all()                        # positive internal energy
        assert U[:, 0].max() > 0.5
        spec = U[:, 6:11].sum(axis=1)
        assert (spec <= rho * (1 + 1e-12)).all()


def _host_ctx(hydro, mesh, rank):
    d = hydro.CudaDevice(hydro.HydroConfig(device_id=-1))
    d.set_mesh(mesh, rank)
    return d


def test_set_mesh_validates_like_mesh_validate(hydro):
    m = hydro.uniform_mesh(2, 2, 2)
    d = hydro.CudaDevice(hydro.HydroConfig(device_id=-1))
    bad = m.neighbor_ids.copy()
    bad[0, 1] = 0
    with pytest.raises(ValueError, match="linked to itself"):
        d.set_mesh(hydro.Mesh(bad, m.pos, m.owner, 1, m.dims))
    bad = m.neighbor_ids.copy()
    bad[0, 1] = 3
    with pytest.raises(ValueError, match="not symmetric"):
        d.set_mesh(hydro.Mesh(bad, m.pos, m.owner, 1, m.dims))
    own = m.owner.copy()
    own[3] = 5
    with pytest.raises(ValueError, match="owner outside the world"):
        d.set_mesh(hydro.Mesh(m.neighbor_ids, m.pos, own, 1, m.dims))
    bad = m.neighbor_ids.copy()
    bad[2, 0] = 99
    with pytest.raises(ValueError, match="out of range"):
        d.set_mesh(hydro.Mesh(bad, m.pos, m.owner, 1, m.dims))


def test_host_only_context_refuses_compute(hydro):
    d = _host_ctx(hydro, hydro.uniform_mesh(2, 2, 2), 0)
    with pytest.raises(hydro.TsError, match="host-only"):
        d.step(1)
    with pytest.raises(hydro.TsError, match="host-only"):
        d.download()


@pytest.mark.parametrize("dims,periodic,world", [((4, 4, 8), "", 2), ((4, 4, 8), "z", 2), ((4, 4, 16), "xyz", 4),
                                                 ((3, 5, 2), "y", 3), ((4, 4, 32), "z", 8),
                                                 # the bench's 8-GPU weak-scaling mesh (8 x Sedov 16^3)
                                                 ((16, 16, 128), "", 8)])
def test_halo_plans_pair_up_across_ranks(hydro, dims, periodic, world):
    """What rank r sends to s is exactly what s expects from r, in the same
    wire order; one aggregated message per directed rank pair."""
    m = hydro.uniform_mesh(*dims, periodic=periodic, world=world)
    ctx = [_host_ctx(hydro, m, r) for r in range(world)]
    total = 0
    for r in range(world):
        owned, n_proxy, n_interior = ctx[r].local_counts()
        assert owned == (m.owner == r).sum()
        for s in range(world):
            if s == r:
                continue
            send, _ = ctx[r].halo_plan(s)
            _, recv = ctx[s].halo_plan(r)
            assert np.array_equal(send, recv)
            for gid, face in send:
                assert m.owner[gid] == r and m.owner[m.neighbor_ids[gid, face]] == s
            total += len(send)
    # every cross-rank directed face link carries exactly one slab
    nb = m.neighbor_ids
    cross = sum(1 for g in range(m.n) for f in range(6) if nb[g, f] >= 0 and m.owner[nb[g, f]] != m.owner[g])
    assert total == cross


def test_interior_boundary_split(hydro):
    m = hydro.uniform_mesh(4, 4, 8, world=2)
    d = _host_ctx(hydro, m, 0)
    owned, proxy, interior = d.local_counts()
    assert (owned, proxy) == (64, 16)   # z-slab split: one 4x4 face of proxies
    assert interior == 48


def test_parse_workload_config_mirrors_reference_rules(hydro):
    cfg = hydro.parse_workload_config("# sedov\nnx=16\nny = 16\nnz=16\nsteps=10\nproblem=sedov\n"
                                      "comm_mode=remote_action\nrecon=minmod\nperiodic=xz\nlevels=3\n")
    assert (cfg.nx, cfg.ny, cfg.nz, cfg.step.num_steps, cfg.problem) == (16, 16, 16, 10, "sedov")
    assert cfg.step.comm_mode == "remote_action" and cfg.recon == "minmod" and cfg.periodic == "xz"
    with pytest.raises(RuntimeError, match="line 2: unknown key 'bogus'"):
        hydro.parse_workload_config("nx=4\nbogus=1\n")
    with pytest.raises(RuntimeError, match="line 1: bad value 'x4' for key 'nx'"):
        hydro.parse_workload_config("nx=x4\n")
    with pytest.raises(RuntimeError, match="line 1: expected key=value"):
        hydro.parse_workload_config("nx\n")
    with pytest.raises(RuntimeError, match="unknown comm mode"):
        hydro.parse_workload_config("comm_mode=carrier_pigeon\n")
    with pytest.raises(RuntimeError, match="N must be 8"):
        hydro.parse_workload_config("N=16\n")
    with pytest.raises(RuntimeError, match="hydro_iterations_per_step must be 3"):
        hydro.parse_workload_config("hydro_iterations=2\n")


def test_invalid_configs_are_rejected(hydro):
    for kw in ({"cells_per_edge": 16}, {"n_species": 9}, {"gamma": 1.0}, {"cfl": 0.0}, {"stream_count": 1}):
        with pytest.raises(ValueError):
            hydro.CudaDevice(hydro.HydroConfig(device_id=-1, **kw))


def test_native_driver_parses_config_like_the_reference(hydro, tmp_path):
    """tools/ts_hydro_run (C++ host over the C ABI) rejects unknown keys with the
    line number, exit code 2 (the reference CLI's usage-error code)."""
    import subprocess
    exe = os.path.join(ROOT, "tools", "ts_hydro_run")
    if not os.path.exists(exe):
        pytest.skip("driver not built")
    bad = tmp_path / "bad.cfg"
    bad.write_text("nx=4\nbogus=1\n")
    r = subprocess.run([exe, str(bad)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 2 and "line 2: unknown key 'bogus'" in r.stderr
