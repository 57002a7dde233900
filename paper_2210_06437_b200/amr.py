"""Coarse-fine AMR meshes for the hydro path.

The reference builds a multi-level octree (``build_mesh``, workload.cpp:264-327)
whose refined parents stay in the sub-grid list and whose ghost links join
same-level faces only (``Mesh::validate``, workload.cpp:160-161).  Octo-Tiger
fills the ghosts of a leaf next to another level from that level and corrects
the coarse fluxes there.  ``amr_mesh`` turns an octree refinement
into what ``ts_hydro_set_amr_mesh`` (include/ts_hydro.h) binds:

* the leaves, level-major and Morton-ordered inside a level;
* per leaf and face a neighbour id: a same-level leaf, a proxy sub-grid or -1
  (outflow at the domain boundary);
* the proxies (ids after the leaves): prolongation of a coarse leaf's octant
  (a fine leaf's neighbour position whose parent is a leaf) or restriction of
  the 8 fine leaves of a refined position (a coarse leaf's neighbour);
* the reflux records: per coarse leaf with a refined face neighbour, the 4
  fine leaves behind each such face, by transverse quadrant.

The mesh must be 2:1 balanced across faces (a ``ValueError`` otherwise);
children of a refined neighbour position that do not touch the face may be
refined further.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Iterable, Tuple, Union

import numpy as np

FACE_DIRS = ((-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1))
PROXY_COLS = 11   # ts_amr_proxy: dst, kind, octant, src[8]
REFLUX_COLS = 25  # ts_amr_reflux: coarse, fine[6][4]


def _morton3(x: int, y: int, z: int) -> int:
    k = 0
    for b in range(21):
        k |= ((x >> b) & 1) << (3 * b) | ((y >> b) & 1) << (3 * b + 1) | ((z >> b) & 1) << (3 * b + 2)
    return k


def transverse_axes(axis: int) -> Tuple[int, int]:
    """(a, b) axes of a pencil along `axis`, as in the oracle's pencil_value / the stage kernel."""
    return (1 if axis == 0 else 0), (1 if axis == 2 else 2)


@dataclass
class AmrMesh:
    dims: Tuple[int, int, int]   # level-0 sub-grid counts
    max_level: int
    level: np.ndarray            # int32 [n_leaves], non-decreasing
    pos: np.ndarray              # int32 [n_leaves, 3], sub-grid position at its own level
    nbr: np.ndarray              # int64 [n_leaves, 6]
    level_first: np.ndarray      # int64 [max_level + 2]
    proxies: np.ndarray          # int32 [n_proxy, 11]
    reflux: np.ndarray           # int32 [n_reflux, 25]

    @property
    def n_leaves(self) -> int:
        return len(self.level)

    @property
    def n_proxy(self) -> int:
        return len(self.proxies)

    @property
    def n_total(self) -> int:
        return self.n_leaves + self.n_proxy

    def cell_centres(self, dx: float) -> np.ndarray:
        """[n_leaves, 3, 512] cell-centre coordinates (x fastest), dx = finest level's."""
        i = np.arange(512)
        loc = np.stack([i & 7, (i >> 3) & 7, i >> 6]).astype(np.float64)  # [3, 512]
        h = dx * np.ldexp(1.0, self.max_level - self.level.astype(np.int64))  # [n]
        return (self.pos[:, :, None] * 8.0 + loc[None] + 0.5) * h[:, None, None]

    def cell_volumes(self, dx: float) -> np.ndarray:
        return np.ldexp(1.0, 3 * (self.max_level - self.level.astype(np.int64))) * dx ** 3

    def total_cells(self) -> int:
        return 512 * self.n_leaves


def amr_mesh(nx: int, ny: int, nz: int,
             refine: Union[Callable[[int, Tuple[int, int, int]], bool], Iterable[Tuple[int, int, int, int]]],
             max_level: int = 1) -> AmrMesh:
    """Leaves of the octree over an nx*ny*nz level-0 box: a position (L, p) with
    L < max_level and refine(L, p) true (or (L, *p) in the given set) is split
    into its 8 children."""
    if not callable(refine):
        marked = {tuple(int(v) for v in r) for r in refine}
        pred = lambda L, p: (L, *p) in marked  # noqa: E731
    else:
        pred = refine
    leaves = []

    def visit(L, p):
        if L < max_level and pred(L, p):
            for o in range(8):
                visit(L + 1, (2 * p[0] + (o & 1), 2 * p[1] + ((o >> 1) & 1), 2 * p[2] + ((o >> 2) & 1)))
        else:
            leaves.append((L, p))

    for z in range(nz):
        for y in range(ny):
            for x in range(nx):
                visit(0, (x, y, z))
    used = max(L for L, _ in leaves)
    leaves.sort(key=lambda e: (e[0], _morton3(*e[1])))
    index = {e: i for i, e in enumerate(leaves)}
    n = len(leaves)
    nbr = np.full((n, 6), -1, np.int64)
    proxies, proxy_of = [], {}
    reflux = {}

    def inside(L, q):
        return 0 <= q[0] < (nx << L) and 0 <= q[1] < (ny << L) and 0 <= q[2] < (nz << L)

    def children(L, q):
        return [(L + 1, (2 * q[0] + (o & 1), 2 * q[1] + ((o >> 1) & 1), 2 * q[2] + ((o >> 2) & 1)))
                for o in range(8)]

    for i, (L, p) in enumerate(leaves):
        for f, d in enumerate(FACE_DIRS):
            q = (p[0] + d[0], p[1] + d[1], p[2] + d[2])
            if not inside(L, q):
                continue
            if (L, q) in index:
                nbr[i, f] = index[(L, q)]
                continue
            parent = (L - 1, (q[0] >> 1, q[1] >> 1, q[2] >> 1))
            if L > 0 and parent in index:
                key = (0, L, q)
                if key not in proxy_of:
                    proxy_of[key] = n + len(proxies)
                    octant = (q[0] & 1) | ((q[1] & 1) << 1) | ((q[2] & 1) << 2)
                    proxies.append([proxy_of[key], 0, octant, index[parent]] + [-1] * 7)
                nbr[i, f] = proxy_of[key]
                continue
            kids = children(L, q)
            axis, side = f >> 1, f & 1
            near = [k for o, k in enumerate(kids) if ((o >> axis) & 1) == (0 if side == 1 else 1)]
            if all(k in index for k in near):
                key = (1, L, q)
                if key not in proxy_of:
                    # children away from this face may be refined further (2:1
                    # holds across faces); the stage kernel reads only the 3
                    # coarse layers next to the face, i.e. the near children,
                    # so a non-leaf child's octant is filled from any leaf child
                    # (never read)
                    first_leaf = next(index[k] for k in kids if k in index)
                    proxy_of[key] = n + len(proxies)
                    proxies.append([proxy_of[key], 1, 0] + [index.get(k, first_leaf) for k in kids])
                nbr[i, f] = proxy_of[key]
                ta, tb = transverse_axes(axis)
                rec = reflux.setdefault(i, [[-1] * 4 for _ in range(6)])
                for qa in range(2):
                    for qb in range(2):
                        off = [0, 0, 0]
                        off[axis] = 0 if side == 1 else 1
                        off[ta], off[tb] = qa, qb
                        rec[f][qa + 2 * qb] = index[(L + 1, tuple(2 * q[k] + off[k] for k in range(3)))]
                continue
            raise ValueError(f"mesh is not 2:1 balanced at leaf {i} (level {L}, {p}) face {f}")

    level = np.array([L for L, _ in leaves], np.int32)
    pos = np.array([p for _, p in leaves], np.int32).reshape(n, 3)
    level_first = np.searchsorted(level, np.arange(used + 2)).astype(np.int64)
    prox = np.array(proxies, np.int32).reshape(-1, PROXY_COLS)
    refl = np.array([[g] + [v for face in rec for v in face] for g, rec in sorted(reflux.items())],
                    np.int32).reshape(-1, REFLUX_COLS)
    return AmrMesh((nx, ny, nz), used, level, pos, nbr, level_first, prox, refl)


def partition(mesh: AmrMesh, world: int) -> np.ndarray:
    """Owner of every leaf: the reference's deal (build_mesh, workload.cpp:298-323)
    — sort by the Morton key of the position scaled to the finest level,
    coarser first on ties, and hand out contiguous chunks, the first
    n % world ranks one larger."""
    if world < 1:
        raise ValueError("world must be positive")
    shift = mesh.max_level - mesh.level.astype(np.int64)
    keys = [(_morton3(int(p[0]) << int(s), int(p[1]) << int(s), int(p[2]) << int(s)), int(L), i)
            for i, (p, s, L) in enumerate(zip(mesh.pos, shift, mesh.level))]
    keys.sort()
    n = mesh.n_leaves
    owner = np.zeros(n, np.int32)
    base, extra = divmod(n, world)
    cursor = 0
    for r in range(world):
        for _ in range(base + (1 if r < extra else 0)):
            owner[keys[cursor][2]] = r
            cursor += 1
    return owner


def from_reference_mesh(level, pos) -> AmrMesh:
    """The leaves of a reference octree (``build_mesh``, workload.cpp:264-327:
    every existing node, refined parents included, with its level and position
    at that level).  The root is one level-0 sub-grid; a node is refined iff
    its children exist (TreeBuilder::refine creates all 8), and the builder's
    force_exists pass makes every refined node's face neighbours exist
    (workload.cpp:234-248), i.e. the leaves are 2:1 balanced across faces —
    which ``amr_mesh`` checks again."""
    level = np.asarray(level, np.int64)
    pos = np.asarray(pos, np.int64).reshape(-1, 3)
    nodes = {(int(L), tuple(int(v) for v in p)) for L, p in zip(level, pos)}
    refined = set()
    for L, p in nodes:
        if L > 0:
            refined.add((L - 1, p[0] >> 1, p[1] >> 1, p[2] >> 1))
    for L, x, y, z in refined:
        if (L, (x, y, z)) not in nodes:
            raise ValueError(f"node ({L}, {x}, {y}, {z}) has children but does not exist")
    max_level = int(level.max()) if len(level) else 0
    if (0, (0, 0, 0)) not in nodes:
        raise ValueError("the reference octree has one level-0 root at (0, 0, 0)")
    return amr_mesh(1, 1, 1, refined, max_level=max_level)


def ic_blast(mesh: AmrMesh, nf: int, dx: float, gamma: float = 1.4, centre=None, width: float = 0.1,
             amp: float = 4.0, drift=(0.0, 0.0, 0.0)) -> np.ndarray:
    """Smooth pressure / density bump (Gaussian) on a uniform background, with an
    optional uniform drift velocity; [n_total, nf, 512] with zero proxies."""
    xc = mesh.cell_centres(dx)
    ext = np.array(mesh.dims, np.float64) * 8 * dx * (1 << mesh.max_level)
    c = ext / 2 if centre is None else np.asarray(centre, np.float64)
    r2 = ((xc - c[None, :, None]) ** 2).sum(axis=1)
    bump = np.exp(-r2 / (width * width))
    rho = 1.0 + 0.5 * amp * bump
    p = 0.1 + amp * bump
    v = np.asarray(drift, np.float64)
    U = np.zeros((mesh.n_total, nf, 512), np.float64)
    eint = p / (gamma - 1.0)
    U[:mesh.n_leaves, 0] = rho
    for k in range(3):
        U[:mesh.n_leaves, 1 + k] = rho * v[k]
    U[:mesh.n_leaves, 4] = eint + 0.5 * rho * float(v @ v)
    U[:mesh.n_leaves, 5] = eint ** (1.0 / gamma)
    for s in range(6, nf):
        U[:mesh.n_leaves, s] = rho * (bump > 0.5 ** (s - 5))
    return U
