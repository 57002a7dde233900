"""Regenerate the golden vectors drawn from the reference itself.

Runs ONLY in the build container, where /root/reference exists: it compiles
the reference's own core sources (proj/core/src/*.cpp minus export.cpp) into
oracle/_ref/libtaskscope_ref.so via `make -C oracle ref`, calls them through
the C shim oracle/ref_shim.cpp and writes

    tests/golden/reference_vectors.json   mix64 / cell_value / face_cell_index /
                                          build_mesh ownership
    tests/golden/reference_ghosts.npz     one ghost-exchange round per comm mode
                                          on hand-built uniform meshes

The GPU box never reads /root/reference: tests use these committed files.

    python tests/golden/gen_golden.py
"""
from __future__ import annotations

import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# (nx, ny, nz, periodic, world) hand-built uniform meshes, plus the row mesh
# of the reference's own tests (test_workload.cpp:38-54): 8 in a row, split 4/4.
GHOST_MESHES = [
    (4, 4, 4, (False, False, False), 1),
    (4, 4, 4, (False, False, False), 3),
    (2, 2, 2, (True, True, True), 2),
    (8, 1, 1, (False, False, False), 2),
]
STEPS = [3]


def main() -> int:
    if not oracle.build_ref():
        print("reference sources not available; nothing regenerated")
        return 1
    R = oracle.ref()
    vec = {"source": "oracle/_ref/libtaskscope_ref.so built from /root/reference/proj/core/src"}
    xs = [0, 1, 2, 3, 7, 11, 0x9E3779B97F4A7C15, 2**63 + 5, 2**64 - 1, 2210, 123456789]
    vec["mix64"] = [[x, R.ref_mix64(x)] for x in xs]
    vec["mix64_2"] = [[a, b, R.ref_mix64_2(a, b)] for a in xs[:6] for b in xs[:6]]
    cv = []
    for g in (0, 1, 5, 63, 4095, 262143):
        for s in (0, 1, 2210):
            for i in (0, 1, 511, 512, 5 * 512 + 17, 10 * 512 + 511):
                cv.append([g, s, i, R.ref_cell_value(g, s, i).hex()])
    vec["cell_value"] = cv
    fci = []
    for edge in (4, 8):
        for face in range(6):
            fci.append([edge, face, [R.ref_face_cell_index(edge, face, j) for j in range(edge * edge)]])
    vec["face_cell_index"] = fci
    meshes = []
    for levels, world, seed in ((2, 1, 3), (2, 2, 1), (3, 3, 7), (4, 4, 0)):
        n = R.ref_build_mesh(levels, world, seed, None, None, None, None, 0)
        owner = np.zeros(n, np.int32)
        level = np.zeros(n, np.int32)
        pos = np.zeros((n, 3), np.int32)
        nbr = np.zeros((n, 6), np.int64)
        i32p = ctypes.POINTER(ctypes.c_int32)
        R.ref_build_mesh(levels, world, seed, owner.ctypes.data_as(i32p), level.ctypes.data_as(i32p),
                         pos.ctypes.data_as(i32p), nbr.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), n)
        kind = np.zeros(n, np.int32)
        R.ref_gravity_kinds(levels, world, seed, kind.ctypes.data_as(i32p), n)
        meshes.append({"levels": levels, "world": world, "seed": seed, "owner": owner.tolist(),
                       "level": level.tolist(), "pos": pos.tolist(), "nbr": nbr.tolist(),
                       "gravity_kind": kind.tolist()})
    vec["build_mesh"] = meshes
    with open(os.path.join(OUT, "reference_vectors.json"), "w") as f:
        json.dump(vec, f, indent=0)

    arrays = {}
    f64p = ctypes.POINTER(ctypes.c_double)
    for k, (nx, ny, nz, per, world) in enumerate(GHOST_MESHES):
        nbr, pos, owner = oracle.uniform_mesh(nx, ny, nz, per, world)
        if (nx, ny, nz) == (8, 1, 1):
            owner = (np.arange(8) >= 4).astype(np.int32)
        n = len(owner)
        arrays[f"m{k}_nbr"] = nbr
        arrays[f"m{k}_pos"] = pos
        arrays[f"m{k}_owner"] = owner
        for step in STEPS:
            cells = np.zeros((n, 512), np.float64)
            R.ref_fill_cells(n, step, cells.ctypes.data_as(f64p))
            ghosts = []
            for mode in (0, 1):
                ghost = np.zeros((n, 6, 64), np.float64)
                parcels = ctypes.c_uint64()
                rc = R.ref_exchange_ghosts(n, nbr.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                           pos.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                           owner.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), world, mode, step,
                                           ghost.ctypes.data_as(f64p), ctypes.byref(parcels))
                assert rc == 0, "reference exchange failed"
                ghosts.append(ghost)
                arrays[f"m{k}_s{step}_mode{mode}_parcels"] = np.array([parcels.value], np.uint64)
            # the reference's own invariant (test_workload.cpp:317-331): both modes agree bitwise
            assert np.array_equal(ghosts[0], ghosts[1])
            arrays[f"m{k}_s{step}_ghost"] = ghosts[0]
    arrays["meshes"] = np.array([[nx, ny, nz, int(p[0]), int(p[1]), int(p[2]), w]
                                 for nx, ny, nz, p, w in GHOST_MESHES], np.int64)
    np.savez_compressed(os.path.join(OUT, "reference_ghosts.npz"), **arrays)
    print("wrote", os.listdir(OUT))
    return 0


if __name__ == "__main__":
    sys.exit(main())
