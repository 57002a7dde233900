"""GPU parity of the coarse-fine AMR path: ts_hydro_set_amr_mesh
+ ts_hydro_step through the C ABI against the oracle's orc_run_amr on the same
inputs.  The proxy fill and reflux kernels follow the oracle operation for
operation and the stage kernel is the uniform path's (bitwise to the oracle),
so the contract is bitwise; RTOL (1e-12, north_star) is the stated tolerance."""
import numpy as np
import pytest

from paper_2210_06437_b200 import amr

pytestmark = pytest.mark.gpu

RTOL = 1e-12
DX = 1.0 / 64
L_SHAPE = {(0, 1, 1, 1), (0, 2, 1, 1), (0, 1, 2, 1), (0, 1, 1, 2), (0, 2, 2, 2)}
CENTRE_BLOCK6 = {(0, x, y, z) for x in (2, 3) for y in (2, 3) for z in (2, 3)}


def gpu_run(hydro, mesh, U0, steps, **kw):
    d = hydro.CudaDevice(hydro.HydroConfig(dx=DX, **kw))
    d.set_amr_mesh(mesh)
    d.upload(U0[:mesh.n_leaves])
    d.step(steps)
    d.synchronize()
    U = d.download()
    dt = d.last_dt()
    recs = d.flush_activity()
    d.close()
    return U, dt, recs


def check(U, ref, n_leaves):
    ref = ref[:n_leaves]
    for f in range(ref.shape[1]):
        scale = np.abs(ref[:, f]).max() or 1.0
        assert np.abs(U[:, f] - ref[:, f]).max() / scale <= RTOL, f
    return np.array_equal(U, ref)


@pytest.mark.parametrize("recon", [0, 1], ids=["ppm", "minmod"])
@pytest.mark.parametrize("species", [0, 5])
@pytest.mark.parametrize("case", ["lshape", "centre6"])
def test_amr_steps_match_oracle_bitwise(hydro, oracle_lib, recon, species, case):
    if case == "lshape":
        m = amr.amr_mesh(4, 4, 4, L_SHAPE)
        centre = (0.625, 0.625, 0.5)
    else:
        m = amr.amr_mesh(6, 6, 6, CENTRE_BLOCK6)
        centre = (1.0, 0.75, 0.75)
    nf = 6 + species
    U0 = amr.ic_blast(m, nf, DX, width=0.06, centre=centre, drift=(0.3, -0.1, 0.2))
    p = oracle_lib.params(nf=nf, recon=recon, dx=DX)
    ref, dts = oracle_lib.run_amr(p, m, U0, 4)
    U, dt, _ = gpu_run(hydro, m, U0, 4, n_species=species, recon=("ppm", "minmod")[recon])
    assert dt == dts[-1]
    assert check(U, ref, m.n_leaves), "AMR path is not bitwise equal to the oracle"


@pytest.mark.parametrize("mode", ["default", "split", "fullfill"])
@pytest.mark.parametrize("recon", [0, 1], ids=["ppm", "minmod"])
def test_three_level_amr_matches_oracle_bitwise(hydro, oracle_lib, recon, mode, monkeypatch):
    """Levels 0-2 (restrictions whose far children are refined further), 3
    steps; one stage launch over all levels and proxies filled only in the
    face layers read (default), one stage launch per level
    (TS_HYDRO_AMR_SPLIT=1), whole proxies filled (TS_HYDRO_AMR_FULLFILL=1)."""
    if mode == "split":
        monkeypatch.setenv("TS_HYDRO_AMR_SPLIT", "1")
    if mode == "fullfill":
        monkeypatch.setenv("TS_HYDRO_AMR_FULLFILL", "1")
    ref = lambda L, p: (L == 0 and all(1 <= v <= 2 for v in p)) or (L == 1 and all(3 <= v <= 4 for v in p))  # noqa
    m = amr.amr_mesh(4, 4, 4, ref, max_level=2)
    dx = DX / 2
    U0 = amr.ic_blast(m, 6, dx, width=0.06, centre=(0.45, 0.5, 0.55), drift=(0.2, 0.1, -0.3))
    p = oracle_lib.params(nf=6, recon=recon, dx=dx)
    ref_U, dts = oracle_lib.run_amr(p, m, U0, 3)
    d = hydro.CudaDevice(hydro.HydroConfig(dx=dx, recon=("ppm", "minmod")[recon]))
    d.set_amr_mesh(m)
    d.upload(U0[:m.n_leaves])
    d.step(3)
    d.synchronize()
    U = d.download()
    assert d.last_dt() == dts[-1]
    d.close()
    assert check(U, ref_U, m.n_leaves)


def test_amr_reflux_conserves_on_gpu(hydro, oracle_lib):
    m = amr.amr_mesh(6, 6, 6, CENTRE_BLOCK6)
    U0 = amr.ic_blast(m, 6, DX, width=0.04, centre=(1.0, 0.75, 0.75))
    vol = m.cell_volumes(DX)
    U, _, _ = gpu_run(hydro, m, U0, 5)
    t0 = np.array([(U0[:m.n_leaves, f].sum(axis=1) * vol).sum() for f in range(5)])
    t1 = np.array([(U[:, f].sum(axis=1) * vol).sum() for f in range(5)])
    assert (np.abs(t1 - t0) / np.abs(t0).max()).max() < 1e-14


def test_amr_free_stream_is_exact_on_gpu(hydro):
    m = amr.amr_mesh(4, 4, 4, L_SHAPE)
    U0 = amr.ic_blast(m, 6, DX, amp=0.0, drift=(0.5, -0.25, 0.125))
    U, _, _ = gpu_run(hydro, m, U0, 3)
    for f in range(6):
        assert (U[:, f] == U0[0, f, 0]).all(), f


def test_amr_medium_mesh_matches_oracle(hydro, oracle_lib):
    """16^3 level-0 box with a refined 4^3 centre: 4544 leaves, 3 steps."""
    m = amr.amr_mesh(16, 16, 16, lambda L, p: all(6 <= v < 10 for v in p))
    assert m.n_leaves == 4096 - 64 + 512
    U0 = amr.ic_blast(m, 6, DX / 2, width=0.2, centre=(1.0, 1.0, 1.0))
    p = oracle_lib.params(nf=6, dx=DX / 2)
    ref, dts = oracle_lib.run_amr(p, m, U0, 3)
    d = hydro.CudaDevice(hydro.HydroConfig(dx=DX / 2))
    d.set_amr_mesh(m)
    d.upload(U0[:m.n_leaves])
    d.step(3)
    d.synchronize()
    U = d.download()
    assert d.last_dt() == dts[-1]
    d.close()
    assert check(U, ref, m.n_leaves)


def test_amr_activity_records_and_refusals(hydro, tmp_path, monkeypatch):
    m = amr.amr_mesh(4, 4, 4, L_SHAPE)
    U0 = amr.ic_blast(m, 6, DX)
    _, _, recs = gpu_run(hydro, m, U0, 2)
    names = [r.name for r in recs]
    # per step: 3 x (fill + one stage launch over both levels + reflux)
    assert names.count("amr_ghost_fill_kernel") == 6
    assert names.count("amr_reflux_kernel") == 6
    assert sum(n.startswith("hydro_stage") for n in names) == 6
    monkeypatch.setenv("TS_HYDRO_AMR_SPLIT", "1")
    _, _, recs = gpu_run(hydro, m, U0, 2)
    # split: one stage launch per level
    assert sum(r.name.startswith("hydro_stage") for r in recs) == 12
    monkeypatch.delenv("TS_HYDRO_AMR_SPLIT")
    for r in recs:
        assert r.start_ns <= r.end_ns
    d = hydro.CudaDevice(hydro.HydroConfig(dx=DX))
    d.set_amr_mesh(m)
    d.upload(U0[:m.n_leaves])
    with pytest.raises(hydro.TsError, match="no dt"):  # the drop-in step needs a dt first, as on uniform meshes
        d.launch_stage(1, [0])
    d.close()


def test_amr_step_host_matches_resident_step(hydro):
    import ctypes
    m = amr.amr_mesh(4, 4, 4, L_SHAPE)
    U0 = amr.ic_blast(m, 6, DX, drift=(0.1, 0.2, 0.3))
    ref, _, _ = gpu_run(hydro, m, U0, 2)
    d = hydro.CudaDevice(hydro.HydroConfig(dx=DX))
    d.set_amr_mesh(m)
    nbytes = m.n_leaves * 6 * 512 * 8
    hin, hout = d.host_pinned_alloc(nbytes), d.host_pinned_alloc(nbytes)
    ctypes.memmove(hin, np.ascontiguousarray(U0[:m.n_leaves]).ctypes.data, nbytes)
    d.step_host(hin, hout, 2)
    out = np.empty((m.n_leaves, 6, 512))
    ctypes.memmove(out.ctypes.data, hout, nbytes)
    d.host_pinned_free(hin)
    d.host_pinned_free(hout)
    d.close()
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("species,recon", [(0, 0), (5, 0), (0, 1)])
def test_amr_on_reference_build_mesh_octrees_matches_oracle(hydro, oracle_lib, golden, species, recon):
    """The AMR path on the reference's own octrees (build_mesh golden meshes,
    levels 3 and 4: 29 and 288 leaves on 3 and 4 levels, 2:1 balanced by the
    reference's TreeBuilder), a drifting blast across every coarse-fine face,
    4 steps: bitwise equal to the oracle."""
    vec, _ = golden
    for m in vec["build_mesh"]:
        if m["levels"] < 3:
            continue
        a = amr.from_reference_mesh(m["level"], m["pos"])
        dx = 1.0 / (8 << a.max_level)
        nf = 6 + species
        U0 = amr.ic_blast(a, nf, dx, width=0.12, centre=(0.4, 0.55, 0.5), drift=(0.3, -0.1, 0.2))
        ref, dts = oracle_lib.run_amr(oracle_lib.params(nf=nf, recon=recon, dx=dx), a, U0, 4)
        d = hydro.CudaDevice(hydro.HydroConfig(dx=dx, n_species=species, recon=("ppm", "minmod")[recon]))
        d.set_amr_mesh(a)
        d.upload(U0[:a.n_leaves])
        d.step(4)
        d.synchronize()
        U = d.download()
        dt = d.last_dt()
        d.close()
        assert dt == dts[-1]
        assert check(U, ref, a.n_leaves), f"levels={m['levels']}: not bitwise equal to the oracle"


def test_amr_checkpoint_restart_is_a_bitwise_continuation(hydro, tmp_path):
    """Persisted state on an AMR mesh (§8(f) rank 4 x rank 2): the checkpoint
    carries the global leaf table (links incl. proxy ids) and the leaf states;
    a fresh context bound to the same AMR mesh restores it and continues
    bitwise equal to the uninterrupted run."""
    m = amr.amr_mesh(4, 4, 4, L_SHAPE)
    U0 = amr.ic_blast(m, 6, DX, width=0.06, centre=(0.625, 0.625, 0.5), drift=(0.3, -0.1, 0.2))
    want, _, _ = gpu_run(hydro, m, U0, 4)
    d = hydro.CudaDevice(hydro.HydroConfig(dx=DX))
    d.set_amr_mesh(m)
    d.upload(U0[:m.n_leaves])
    d.step(2)
    path = str(tmp_path / "amr.ckpt")
    d.save(path)
    d.close()
    r = hydro.CudaDevice(hydro.HydroConfig(dx=DX))
    r.set_amr_mesh(m)
    r.restore([path])
    r.step(2)
    got = r.download()
    r.close()
    assert np.array_equal(got, want)


@pytest.mark.parametrize("order", ["stage", "grid"])
def test_amr_dropin_steps_match_batched_bitwise(hydro, golden, order):
    """The per-sub-grid drop-in on AMR meshes (an L-shaped refinement and the
    reference's own 4-level build_mesh octree): every leaf's stage launched
    alone on a rotating stream in a scrambled order — the proxy fill and the
    reflux between the stages come in behind every leaf's previous stage —
    bitwise equal to the batched AMR steps, equal dt."""
    vec, _ = golden
    ref_mesh = max(vec["build_mesh"], key=lambda e: len(e["level"]))
    cases = [(amr.amr_mesh(4, 4, 4, L_SHAPE), DX, (0.625, 0.625, 0.5)),
             (amr.from_reference_mesh(ref_mesh["level"], ref_mesh["pos"]), None, (0.4, 0.55, 0.5))]
    for m, dx, centre in cases:
        dx = dx or 1.0 / (8 << m.max_level)
        U0 = amr.ic_blast(m, 6, dx, width=0.08, centre=centre, drift=(0.3, -0.1, 0.2))
        r = hydro.CudaDevice(hydro.HydroConfig(dx=dx))
        r.set_amr_mesh(m)
        r.upload(U0[:m.n_leaves])
        r.step(3)
        want, dt_want = r.download(), r.last_dt()
        r.close()
        d = hydro.CudaDevice(hydro.HydroConfig(dx=dx))
        d.set_amr_mesh(m)
        d.upload(U0[:m.n_leaves])
        d.compute_dt()
        n = m.n_leaves
        for step in range(3):
            perm = [(k * 37 + step * 11 + 5) % n for k in range(n)] if n % 37 else list(range(n))[::-1]
            launches = ([(st, g) for st in (1, 2, 3) for g in perm] if order == "stage"
                        else [(st, g) for g in perm for st in (1, 2, 3)])
            for i, (st, g) in enumerate(launches):
                d.launch_stage(st, [g], stream_id=1 + i % 16, guid=g)
            d.finish_step()
        got, dt = d.download(), d.last_dt()
        names = {r.name for r in d.flush_activity()}
        d.close()
        assert dt == dt_want
        assert np.array_equal(got, want), f"leaves={n}: drop-in differs from the batched AMR steps"
        assert {"amr_ghost_fill_kernel", "amr_reflux_kernel", "hydro_stage3_kernel"} <= names
