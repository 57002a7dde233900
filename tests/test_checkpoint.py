"""Persisted state format: checkpoint files through the
C ABI (ts_hydro_checkpoint_{write,info,read}).  Host-only: no GPU needed.
The GPU restart / offline-parity tests are in test_gpu.py."""
import struct

import numpy as np
import pytest

NC = 512


def _state(rng, n, nf):
    return rng.standard_normal((n, nf, NC))


@pytest.mark.parametrize("species", [0, 5])
def test_write_read_round_trip(hydro, tmp_path, species):
    rng = np.random.default_rng(7)
    m = hydro.uniform_mesh(3, 2, 4, periodic="y", world=2)
    cfg = hydro.HydroConfig(n_species=species, dx=1 / 24, recon="minmod")
    gids = m.owned_by(1)
    st = _state(rng, gids.size, cfg.nf)
    p = str(tmp_path / "r1.tsh")
    hydro.write_checkpoint(p, cfg, m, gids, st, steps_done=17, rank=1)
    ck = hydro.read_checkpoint(p)
    h = ck.header
    assert (h["version"], h["nf"], h["n_species"], h["recon"], h["cells_per_edge"]) == (1, cfg.nf, species, 1, 8)
    assert (h["gamma"], h["cfl"], h["dx"], h["p_floor"]) == (cfg.gamma, cfg.cfl, cfg.dx, cfg.p_floor)
    assert (h["n_grids"], h["n_records"], h["steps_done"], h["world"], h["rank"]) == (m.n, gids.size, 17, 2, 1)
    assert np.array_equal(ck.neighbor_ids, m.neighbor_ids)
    assert np.array_equal(ck.owner, m.owner)
    assert np.array_equal(ck.global_ids, gids)
    assert np.array_equal(ck.state, st)


def test_layout_matches_the_documented_format(hydro, tmp_path):
    """An independent reader of the layout documented in ts_hydro_ckpt.cpp."""
    rng = np.random.default_rng(3)
    m = hydro.uniform_mesh(2, 2, 2)
    cfg = hydro.HydroConfig(dx=0.0625)
    gids = np.array([5, 1, 6])
    st = _state(rng, 3, 6)
    p = tmp_path / "a.tsh"
    hydro.write_checkpoint(str(p), cfg, m, gids, st, steps_done=3)
    raw = p.read_bytes()
    assert raw[:8] == b"TSHYDRO\0"
    version, hbytes, nf, ns, recon, cpe = struct.unpack_from("<IIiiii", raw, 8)
    assert (version, hbytes, nf, ns, recon, cpe) == (1, 128, 6, 0, 0, 8)
    assert struct.unpack_from("<dddd", raw, 32) == (1.4, 0.4, 0.0625, 1e-12)
    n_grids, n_rec, steps = struct.unpack_from("<qqQ", raw, 64)
    assert (n_grids, n_rec, steps) == (8, 3, 3)
    checksum = struct.unpack_from("<Q", raw, 96)[0]
    payload = raw[128:]
    h = 0xcbf29ce484222325
    for b in payload:
        h = ((h ^ b) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    assert h == checksum
    o = 0
    nbr = np.frombuffer(payload, np.int64, 8 * 6, o).reshape(8, 6)
    o += 8 * 6 * 8
    own = np.frombuffer(payload, np.int32, 8, o)
    o += 8 * 4
    gid = np.frombuffer(payload, np.int64, 3, o)
    o += 3 * 8
    s = np.frombuffer(payload, np.float64, 3 * 6 * NC, o).reshape(3, 6, NC)
    assert o + s.nbytes == len(payload)
    assert np.array_equal(nbr, m.neighbor_ids) and np.array_equal(own, m.owner)
    assert np.array_equal(gid, gids) and np.array_equal(s, st)


def test_corrupt_truncated_or_foreign_files_are_rejected(hydro, tmp_path):
    m = hydro.uniform_mesh(2, 1, 1)
    cfg = hydro.HydroConfig()
    p = tmp_path / "c.tsh"
    hydro.write_checkpoint(str(p), cfg, m, [0, 1], np.ones((2, 6, NC)))
    good = p.read_bytes()
    hydro.read_checkpoint(str(p))
    bad = bytearray(good)
    bad[200] ^= 1  # one payload bit
    p.write_bytes(bytes(bad))
    with pytest.raises(ValueError):
        hydro.read_checkpoint(str(p))
    p.write_bytes(good[:-8])  # truncated
    with pytest.raises(ValueError):
        hydro.read_checkpoint(str(p))
    p.write_bytes(good + b"\0")  # trailing bytes
    with pytest.raises(ValueError):
        hydro.read_checkpoint(str(p))
    p.write_bytes(b"XSHYDRO\0" + good[8:])  # magic
    with pytest.raises(ValueError):
        hydro.read_checkpoint(str(p))
    with pytest.raises(ValueError):
        hydro.read_checkpoint(str(tmp_path / "missing.tsh"))


def test_write_rejects_bad_arguments(hydro, tmp_path):
    m = hydro.uniform_mesh(2, 1, 1)
    cfg = hydro.HydroConfig()
    with pytest.raises(ValueError):  # shape
        hydro.write_checkpoint(str(tmp_path / "x"), cfg, m, [0], np.ones((2, 6, NC)))
    with pytest.raises(ValueError):  # global id outside the mesh
        hydro.write_checkpoint(str(tmp_path / "x"), cfg, m, [2], np.ones((1, 6, NC)))
    with pytest.raises(ValueError):  # unwritable path
        hydro.write_checkpoint(str(tmp_path / "no" / "such" / "dir"), cfg, m, [0], np.ones((1, 6, NC)))
