"""Python mirror of the reference's workload interface over libts_hydro.so.

The reference (``taskscope``) drives the hydro path through
``WorkloadSession`` (proj/core/include/taskscope/workload.hpp:165-214) on a
``Mesh`` of ``SubGrid``s (workload.hpp:53-97), with the device behind
``SimDevice`` (device.hpp:45-119).  This module keeps those names and their
argument meaning and error behaviour so tests read like the reference's own:

    mesh    = uniform_mesh(4, 4, 4)                 # Mesh (hand-built, Morton-numbered)
    device  = CudaDevice(HydroConfig(dx=1/32))      # SimDevice's role, real B200
    session = WorkloadSession(mesh, device, StepConfig(num_steps=10))
    session.load_problem("sod")
    point   = session.run_benchmark()               # ScalingPoint(cells_per_second=...)

Everything computes in ``libts_hydro.so`` (C ABI: include/ts_hydro.h).  There
is no CPU fallback: if the library is missing or the GPU call fails, the call
raises.
"""
from __future__ import annotations

import ctypes
import dataclasses
import io
import os
import time
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TS_HYDRO_LIB") or os.path.join(HERE, "libts_hydro.so")
HEADER_PATH = os.path.join(os.path.dirname(HERE), "include", "ts_hydro.h")

N = 8
NC = 512

TS_OK, TS_EINVAL, TS_ESHUTDOWN, TS_ECUDA, TS_ENCCL, TS_ENOMEM, TS_ESTATE, TS_ECOMM = range(8)
RECON = {"ppm": 0, "minmod": 1}
PROBLEMS = {"sod": 0, "sedov": 1, "random": 2, "polytrope": 3, "binary": 4}
ACTIVITY_KINDS = ("kernel", "copy_host_to_device", "copy_device_to_host", "copy_device_to_device",
                  "alloc", "free")

# Reference task / kernel taxonomy (workload.hpp:32-48).
kTaskExecuteStep = "execute_step"
kTaskCollectHydroBoundaries = "collect_hydro_boundaries"
kTaskComputeFluxes = "compute_fluxes"
kKernelReconstruct = "reconstruct_kernel"
kKernelFlux = "flux_kernel"


# TS_HYDRO_CHECK_STRICT with a TS_CHECK library: failures recorded by devices
# at close (tests/conftest.py asserts it stays empty after every test)
CHECK_FAILURES: list = []


class TsError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class _Config(ctypes.Structure):
    _fields_ = [
        ("device_id", ctypes.c_int32),
        ("stream_count", ctypes.c_uint32),
        ("activity_buffer_capacity", ctypes.c_uint32),
        ("cells_per_edge", ctypes.c_int32),
        ("n_species", ctypes.c_int32),
        ("recon", ctypes.c_int32),
        ("gamma", ctypes.c_double),
        ("cfl", ctypes.c_double),
        ("dx", ctypes.c_double),
        ("p_floor", ctypes.c_double),
    ]


class _Record(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_uint8),
        ("has_bytes", ctypes.c_uint8),
        ("reserved", ctypes.c_uint16),
        ("device_id", ctypes.c_int32),
        ("stream_id", ctypes.c_int32),
        ("pad", ctypes.c_int32),
        ("name", ctypes.c_char_p),
        ("start_ns", ctypes.c_uint64),
        ("end_ns", ctypes.c_uint64),
        ("bytes", ctypes.c_uint64),
        ("correlation_guid", ctypes.c_uint64),
    ]


class _MemState(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint64) for k in ("current_device_bytes", "peak_device_bytes",
                                               "current_host_pinned_bytes", "peak_host_pinned_bytes")]


class _CkptHeader(ctypes.Structure):
    """ts_hydro_checkpoint_header (ts_hydro.h)."""
    _fields_ = [("version", ctypes.c_uint32), ("nf", ctypes.c_int32), ("n_species", ctypes.c_int32),
                ("recon", ctypes.c_int32), ("cells_per_edge", ctypes.c_int32), ("gamma", ctypes.c_double),
                ("cfl", ctypes.c_double), ("dx", ctypes.c_double), ("p_floor", ctypes.c_double),
                ("n_grids", ctypes.c_int64), ("n_records", ctypes.c_int64), ("steps_done", ctypes.c_uint64),
                ("world", ctypes.c_int32), ("rank", ctypes.c_int32), ("checksum", ctypes.c_uint64)]


_lib = None
_vp = ctypes.c_void_p
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_f64p = ctypes.POINTER(ctypes.c_double)
_u64p = ctypes.POINTER(ctypes.c_uint64)
DONE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p)
SINK_FN = ctypes.CFUNCTYPE(None, ctypes.POINTER(_Record), ctypes.c_uint64, ctypes.c_void_p)

_SIGNATURES = {
    "ts_hydro_abi_version": (ctypes.c_int, []),
    "ts_hydro_default_config": (None, [ctypes.POINTER(_Config)]),
    "ts_hydro_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "ts_hydro_create": (ctypes.c_int, [ctypes.POINTER(_Config), ctypes.POINTER(_vp)]),
    "ts_hydro_last_error": (ctypes.c_char_p, [_vp]),
    "ts_hydro_shutdown": (ctypes.c_int, [_vp]),
    "ts_hydro_destroy": (ctypes.c_int, [_vp]),
    "ts_hydro_num_fields": (ctypes.c_int, [_vp]),
    "ts_hydro_uniform_mesh": (ctypes.c_int, [ctypes.c_int32] * 5 + [_i64p, _i32p, _i32p]),
    "ts_hydro_set_mesh": (ctypes.c_int, [_vp, ctypes.c_int64, _i64p, _i32p, ctypes.c_int32, ctypes.c_int32]),
    "ts_hydro_set_amr_mesh": (ctypes.c_int, [_vp, ctypes.c_int64, _i64p, _i32p, ctypes.c_int32, ctypes.c_int64,
                                             _i32p, ctypes.c_int64, _i32p]),
    "ts_hydro_set_amr_mesh_partitioned": (ctypes.c_int, [_vp, ctypes.c_int64, _i64p, _i32p, ctypes.c_int32,
                                                         ctypes.c_int64, _i32p, ctypes.c_int64, _i32p, _i32p,
                                                         ctypes.c_int32, ctypes.c_int32]),
    "ts_hydro_local_counts": (ctypes.c_int, [_vp, _i64p, _i64p, _i64p]),
    "ts_hydro_owned_ids": (ctypes.c_int, [_vp, _i64p]),
    "ts_hydro_halo_plan": (ctypes.c_int, [_vp, ctypes.c_int32, _i64p, _i64p, _i64p, _i64p]),
    "ts_hydro_ic_fill": (ctypes.c_int, [ctypes.POINTER(_Config), ctypes.c_int32, ctypes.c_int64, _i64p, _i32p,
                                        _i32p, ctypes.c_uint64, _f64p]),
    "ts_hydro_upload": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int64, _f64p]),
    "ts_hydro_download": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int64, _f64p]),
    "ts_hydro_init_random": (ctypes.c_int, [_vp, ctypes.c_uint64]),
    "ts_hydro_download_buffer": (ctypes.c_int, [_vp, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, _f64p]),
    "ts_hydro_compute_dt": (ctypes.c_int, [_vp, _f64p]),
    "ts_hydro_step": (ctypes.c_int, [_vp, ctypes.c_uint64]),
    "ts_hydro_step_host": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_uint64]),
    "ts_hydro_step_host_async": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_uint64, DONE_FN, _vp]),
    "ts_hydro_synchronize": (ctypes.c_int, [_vp]),
    "ts_hydro_time_steps": (ctypes.c_int, [_vp, ctypes.c_uint64, _f64p]),
    "ts_hydro_last_dt": (ctypes.c_int, [_vp, _f64p]),
    "ts_hydro_steps_done": (ctypes.c_int, [_vp, _u64p]),
    "ts_hydro_launch_count": (ctypes.c_int, [_vp, _u64p]),
    "ts_hydro_launch_stage": (ctypes.c_int, [_vp, ctypes.c_int32, _i64p, ctypes.c_int64, ctypes.c_uint32,
                                             ctypes.c_uint64, DONE_FN, _vp]),
    "ts_hydro_finish_step": (ctypes.c_int, [_vp]),
    "ts_hydro_exchange_faces": (ctypes.c_int, [_vp, _f64p]),
    "ts_hydro_fill_halo": (ctypes.c_int, [_vp, ctypes.c_int32, _f64p]),
    "ts_hydro_nccl_unique_id": (ctypes.c_int, [ctypes.c_char_p]),
    "ts_hydro_comm_init": (ctypes.c_int, [_vp, ctypes.c_char_p, ctypes.c_int32, ctypes.c_int32]),
    "ts_hydro_halo_exchange": (ctypes.c_int, [_vp]),
    "ts_hydro_p2p_blob_size": (ctypes.c_uint64, []),
    "ts_hydro_selftest_math": (ctypes.c_int, [_vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int32, _u64p, _u64p]),
    "ts_hydro_p2p_export": (ctypes.c_int, [_vp, ctypes.c_void_p]),
    "ts_hydro_p2p_import": (ctypes.c_int, [_vp, ctypes.c_char_p, ctypes.c_int32]),
    "ts_hydro_set_activity_sink": (ctypes.c_int, [_vp, SINK_FN, _vp]),
    "ts_hydro_set_profiling": (ctypes.c_int, [_vp, ctypes.c_int32]),
    "ts_hydro_gravity_p2p": (ctypes.c_int, [_vp, ctypes.c_double, ctypes.c_int32, _i64p, ctypes.c_int64,
                                            ctypes.c_uint32, ctypes.c_uint64, DONE_FN, _vp]),
    "ts_hydro_download_gravity": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int64, _f64p]),
    "ts_hydro_set_gravity_tree": (ctypes.c_int, [_vp, ctypes.c_int64, _i32p, _i32p, _i32p, ctypes.c_double]),
    "ts_hydro_gravity_tree": (ctypes.c_int, [ctypes.c_int64, _i32p, _i32p, _i32p, ctypes.c_int64, _i32p, _i32p,
                                             _i32p, _i32p, _i64p]),
    "ts_hydro_gravity_kick": (ctypes.c_int, [_vp, ctypes.c_double]),
    "ts_hydro_step_gravity": (ctypes.c_int, [_vp, ctypes.c_uint64, ctypes.c_double, ctypes.c_int32]),
    "ts_hydro_gravity_fmm": (ctypes.c_int, [_vp, ctypes.c_double, ctypes.c_int32, ctypes.c_uint32, ctypes.c_uint64,
                                            DONE_FN, _vp]),
    "ts_hydro_debug_check": (ctypes.c_int, [_vp, _u64p, ctypes.c_int32]),
    "ts_hydro_check_build": (ctypes.c_int, []),
    "ts_hydro_flush_activity": (ctypes.c_int, [_vp, ctypes.POINTER(_Record), ctypes.c_uint64, _u64p]),
    "ts_hydro_memory_state": (ctypes.c_int, [_vp, ctypes.POINTER(_MemState)]),
    "ts_hydro_clock_ns": (ctypes.c_uint64, []),
    "ts_hydro_host_alloc": (ctypes.c_int, [_vp, ctypes.c_uint64, ctypes.POINTER(_vp)]),
    "ts_hydro_host_free": (ctypes.c_int, [_vp, _vp]),
    "ts_hydro_checkpoint_write": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(_Config), ctypes.c_int64, _i64p,
                                                 _i32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, _i64p,
                                                 _f64p, ctypes.c_uint64]),
    "ts_hydro_checkpoint_info": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(_CkptHeader)]),
    "ts_hydro_checkpoint_read": (ctypes.c_int, [ctypes.c_char_p, _i64p, _i32p, _i64p, _f64p]),
    "ts_hydro_save": (ctypes.c_int, [_vp, ctypes.c_char_p]),
    "ts_hydro_restore": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_char_p), ctypes.c_int32]),
    "ts_hydro_get_mesh": (ctypes.c_int, [_vp, _i64p, _i64p, _i32p, _i32p, _i32p]),
    "ts_hydro_get_config": (ctypes.c_int, [_vp, ctypes.POINTER(_Config)]),
    "ts_hydro_launch_kernel": (ctypes.c_int, [_vp, ctypes.c_char_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64,
                                              DONE_FN, _vp]),
    "ts_hydro_enqueue_copy": (ctypes.c_int, [_vp, ctypes.c_int32, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64,
                                             DONE_FN, _vp]),
    "ts_hydro_device_alloc": (ctypes.c_int, [_vp, ctypes.c_uint64, _u64p]),
    "ts_hydro_device_free": (ctypes.c_int, [_vp, ctypes.c_uint64]),
    "ts_hydro_device_ptr": (ctypes.c_int, [_vp, ctypes.c_uint64, ctypes.POINTER(_vp)]),
    "ts_hydro_debug_cta_log": (ctypes.c_int, [_vp, _u64p, ctypes.c_uint64, _u64p]),
}


def lib():
    """Load libts_hydro.so; raises (never falls back) when it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2210_06437_b200.build` "
                              "(there is no CPU fallback for the hydro path)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


# ---------------------------------------------------------------------------
# Configuration (StepConfig / WorkloadConfig, workload.hpp:114-160)
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class HydroConfig:
    """Device + numerics configuration (DeviceConfig, device.hpp:22-27, plus the hydro knobs)."""
    device_id: int = 0
    stream_count: int = 128
    activity_buffer_capacity: int = 1024
    cells_per_edge: int = 8
    n_species: int = 0
    recon: str = "ppm"
    gamma: float = 1.4
    cfl: float = 0.4
    dx: float = 1.0 / 32
    p_floor: float = 1e-12

    @property
    def nf(self) -> int:
        return 6 + self.n_species

    def to_c(self) -> _Config:
        if self.recon not in RECON:
            raise ValueError(f"unknown reconstruction '{self.recon}'")
        return _Config(self.device_id, self.stream_count, self.activity_buffer_capacity, self.cells_per_edge,
                       self.n_species, RECON[self.recon], self.gamma, self.cfl, self.dx, self.p_floor)


@dataclasses.dataclass
class StepConfig:
    """workload.hpp:114-126. hydro_iterations_per_step is the RK stage count (3)."""
    num_steps: int = 40
    hydro_iterations_per_step: int = 3
    comm_mode: str = "direct_local"
    seed: int = 0

    def validate(self) -> None:
        if self.hydro_iterations_per_step != 3:
            raise ValueError("hydro_iterations_per_step must be 3 (SSP-RK3 stages)")
        if self.comm_mode not in ("remote_action", "direct_local"):
            raise ValueError(f"unknown comm mode '{self.comm_mode}'")


@dataclasses.dataclass
class WorkloadConfig:
    """The key=value benchmark description (workload.hpp:148-154) plus the hydro keys."""
    nx: int = 4
    ny: int = 4
    nz: int = 4
    periodic: str = ""
    cells_per_edge: int = 8
    stream_count: int = 128
    problem: str = "sod"
    species: int = 0
    gamma: float = 1.4
    cfl: float = 0.4
    recon: str = "ppm"
    gpus: int = 1
    step: StepConfig = dataclasses.field(default_factory=StepConfig)


_INT_KEYS = {"nx", "ny", "nz", "N", "streams", "species", "gpus", "steps", "hydro_iterations", "seed",
             "levels", "gravity_iterations", "kernel_min_ns", "kernel_max_ns"}


def parse_workload_config(text: str) -> WorkloadConfig:
    """Mirror of parse_workload_config (workload.cpp:382-432): key=value lines,
    '#' comments, unknown keys and malformed values fail with the line number."""
    cfg = WorkloadConfig()
    for line_no, raw in enumerate(io.StringIO(text), start=1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        if "=" not in line:
            raise RuntimeError(f"workload config line {line_no}: expected key=value")
        key, value = (s.strip() for s in line.split("=", 1))
        if not key:
            raise RuntimeError(f"workload config line {line_no}: empty key")
        try:
            if key in _INT_KEYS:
                if not value.lstrip("-").isdigit():
                    raise ValueError
                iv = int(value)
            if key == "nx":
                cfg.nx = iv
            elif key == "ny":
                cfg.ny = iv
            elif key == "nz":
                cfg.nz = iv
            elif key == "N":
                cfg.cells_per_edge = iv
            elif key == "streams":
                cfg.stream_count = iv
            elif key == "species":
                cfg.species = iv
            elif key == "gpus":
                cfg.gpus = iv
            elif key == "steps":
                cfg.step.num_steps = iv
            elif key == "hydro_iterations":
                cfg.step.hydro_iterations_per_step = iv
            elif key == "seed":
                cfg.step.seed = iv
            elif key in ("levels", "gravity_iterations", "kernel_min_ns", "kernel_max_ns"):
                pass  # reference keys with no meaning for the real hydro path (gravity frozen)
            elif key == "comm_mode":
                if value not in ("remote_action", "direct_local"):
                    raise RuntimeError(f"workload config line {line_no}: unknown comm mode '{value}'")
                cfg.step.comm_mode = value
            elif key == "problem":
                if value not in PROBLEMS:
                    raise RuntimeError(f"workload config line {line_no}: unknown problem '{value}'")
                cfg.problem = value
            elif key == "recon":
                if value not in RECON:
                    raise RuntimeError(f"workload config line {line_no}: unknown recon '{value}'")
                cfg.recon = value
            elif key == "periodic":
                if any(ch not in "xyz" for ch in value):
                    raise ValueError
                cfg.periodic = value
            elif key in ("gamma", "cfl"):
                setattr(cfg, key, float(value))
            else:
                raise RuntimeError(f"workload config line {line_no}: unknown key '{key}'")
        except ValueError:
            raise RuntimeError(f"workload config line {line_no}: bad value '{value}' for key '{key}'") from None
    if min(cfg.nx, cfg.ny, cfg.nz) < 1:
        raise RuntimeError("workload config: mesh extents must be positive")
    if cfg.cells_per_edge != 8:
        raise RuntimeError("workload config: N must be 8")
    if cfg.stream_count < 2:
        raise RuntimeError("workload config: streams must be at least 2")
    try:
        cfg.step.validate()
    except ValueError as e:
        raise RuntimeError(f"workload config: {e}") from None
    return cfg


# ---------------------------------------------------------------------------
# Mesh (workload.hpp:76-103)
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class Mesh:
    """Single-level mesh of 8^3 sub-grids: neighbour table [n][6] (face order
    -x,+x,-y,+y,-z,+z; -1 = domain boundary), positions [n][3], owners [n]."""
    neighbor_ids: np.ndarray
    pos: np.ndarray
    owner: np.ndarray
    world_size: int = 1
    dims: tuple = (1, 1, 1)

    @property
    def n(self) -> int:
        return int(self.neighbor_ids.shape[0])

    def total_cells(self) -> int:
        return self.n * NC

    def owned_by(self, rank: int) -> np.ndarray:
        return np.nonzero(self.owner == rank)[0]

    def neighbor_pairs(self) -> int:
        return int((self.neighbor_ids >= 0).sum()) // 2

    def local_neighbor_pairs(self) -> int:
        nb = self.neighbor_ids
        g = np.repeat(np.arange(self.n), 6).reshape(self.n, 6)
        m = nb >= 0
        return int((self.owner[g[m]] == self.owner[nb[m]]).sum()) // 2


GRAVITY_KINDS = ("multipole_root_kernel", "multipole_kernel", "p2m_kernel", "p2p_kernel")


def gravity_tree(level, pos, dims):
    """The gravity octree of these leaves (ts_hydro_gravity_tree; host only):
    dict of per-node level, pos [n][3], kind (index into GRAVITY_KINDS, the
    reference's gravity_kernel_name choice) and leaf (leaf index or -1)."""
    lv = np.ascontiguousarray(level, np.int32)
    ps = np.ascontiguousarray(np.asarray(pos).reshape(-1, 3), np.int32)
    dm = np.ascontiguousarray(dims, np.int32)
    n = ctypes.c_int64()
    args = (len(lv), _p(lv, _i32p), _p(ps, _i32p), _p(dm, _i32p))
    if lib().ts_hydro_gravity_tree(*args, 0, None, None, None, None, ctypes.byref(n)) != TS_OK:
        raise ValueError("malformed gravity tree (overlapping leaves or positions outside the domain)")
    k = n.value
    lev, kind, leaf = (np.zeros(k, np.int32) for _ in range(3))
    pso = np.zeros((k, 3), np.int32)
    lib().ts_hydro_gravity_tree(*args, k, _p(lev, _i32p), _p(pso, _i32p), _p(kind, _i32p), _p(leaf, _i32p),
                                ctypes.byref(n))
    return {"level": lev, "pos": pso, "kind": kind, "leaf": leaf}


def uniform_mesh(nx: int, ny: int, nz: int, periodic: str = "", world: int = 1, order: str = "morton") -> Mesh:
    """order: "morton" (build_mesh's curve) or "row" (x fastest, z slowest)."""
    if order not in ("morton", "row"):
        raise ValueError(f"unknown mesh order '{order}'")
    n = nx * ny * nz
    nbr = np.zeros((n, 6), np.int64)
    pos = np.zeros((n, 3), np.int32)
    owner = np.zeros(n, np.int32)
    mask = sum(1 << "xyz".index(ch) for ch in periodic) | (8 if order == "row" else 0)
    rc = lib().ts_hydro_uniform_mesh(nx, ny, nz, mask, world, _p(nbr, _i64p), _p(pos, _i32p), _p(owner, _i32p))
    if rc != TS_OK:
        raise ValueError("mesh extents and world size must be positive")
    return Mesh(nbr, pos, owner, world, (nx, ny, nz))


def ic_fill(cfg: HydroConfig, problem: str, mesh: Mesh, grids: Sequence[int], seed: int = 2210) -> np.ndarray:
    """Host initial conditions for the listed global sub-grids ([len][nf][512])."""
    grids = np.ascontiguousarray(np.asarray(grids, np.int64))
    out = np.zeros((len(grids), cfg.nf, NC), np.float64)
    pos = np.ascontiguousarray(mesh.pos[grids], np.int32)
    dims = np.asarray(mesh.dims, np.int32)
    c = cfg.to_c()
    rc = lib().ts_hydro_ic_fill(ctypes.byref(c), PROBLEMS[problem], len(grids), _p(grids, _i64p), _p(pos, _i32p),
                                _p(dims, _i32p), seed, _p(out, _f64p))
    if rc != TS_OK:
        raise ValueError(f"ic_fill failed ({rc})")
    return out


# ---------------------------------------------------------------------------
# Device (SimDevice's role, device.hpp:45-119)
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class ActivityRecord:
    """snapshot.hpp:88-99; timestamps in steady_clock ns."""
    kind: str
    name: str
    device_id: int
    stream_id: int
    start_ns: int
    end_ns: int
    bytes: Optional[int]
    correlation_guid: int


class CudaDevice:
    """One B200 context: buffers, streams, halo plans, timing hook."""

    def __init__(self, config: HydroConfig = None):
        self.config = config or HydroConfig()
        L = lib()
        h = _vp()
        c = self.config.to_c()
        rc = L.ts_hydro_create(ctypes.byref(c), ctypes.byref(h))
        if rc != TS_OK:
            if rc == TS_EINVAL:
                raise ValueError("invalid hydro configuration")
            raise TsError(rc, f"ts_hydro_create failed: {L.ts_hydro_strerror(rc).decode()}")
        self._h = h
        self._callbacks = []
        self._sink = None

    # -- plumbing
    def _check(self, rc: int, what: str) -> None:
        if rc == TS_OK:
            return
        msg = f"{what}: {lib().ts_hydro_last_error(self._h).decode()}"
        if rc == TS_EINVAL:
            raise ValueError(msg)
        if rc == TS_ESHUTDOWN:
            raise RuntimeError(msg)
        raise TsError(rc, msg)

    @property
    def handle(self):
        return self._h

    @property
    def nf(self) -> int:
        return lib().ts_hydro_num_fields(self._h)

    def close(self) -> None:
        if self._h:
            bad = None
            if os.environ.get("TS_HYDRO_CHECK_STRICT") and lib().ts_hydro_check_build():
                try:
                    bad = self.debug_check()
                except Exception:  # e.g. a shut-down device
                    bad = None
            lib().ts_hydro_destroy(self._h)
            self._h = None
            if bad is not None and bad[0] != 0:
                CHECK_FAILURES.append(bad)
                raise AssertionError(f"self-check build recorded {bad[0]} protocol / bounds failures "
                                     f"(first: code {bad[1]}, operands {bad[2]}, {bad[3]}; DESIGN.md section 13)")

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def shutdown(self) -> None:
        self._check(lib().ts_hydro_shutdown(self._h), "shutdown")

    # -- mesh / state
    def set_mesh(self, mesh: Mesh, rank: int = 0) -> None:
        nbr = np.ascontiguousarray(mesh.neighbor_ids, np.int64)
        own = np.ascontiguousarray(mesh.owner, np.int32)
        self._check(lib().ts_hydro_set_mesh(self._h, mesh.n, _p(nbr, _i64p), _p(own, _i32p), mesh.world_size, rank),
                    "set_mesh")
        self.mesh = mesh
        self.rank = rank

    def set_amr_mesh(self, mesh, owner=None, rank: int = 0, world: Optional[int] = None) -> None:
        """Bind a coarse-fine AMR mesh (paper_2210_06437_b200.amr.AmrMesh); with
        owner (per leaf, e.g. amr.partition) the rank's part of a multi-rank run."""
        nbr = np.ascontiguousarray(mesh.nbr, np.int64)
        lev = np.ascontiguousarray(mesh.level, np.int32)
        px = np.ascontiguousarray(mesh.proxies, np.int32)
        rf = np.ascontiguousarray(mesh.reflux, np.int32)
        if owner is None:
            self._check(lib().ts_hydro_set_amr_mesh(self._h, mesh.n_leaves, _p(nbr, _i64p), _p(lev, _i32p),
                                                    mesh.max_level, mesh.n_proxy, _p(px, _i32p), len(rf),
                                                    _p(rf, _i32p)), "set_amr_mesh")
        else:
            own = np.ascontiguousarray(owner, np.int32)
            world = int(own.max()) + 1 if world is None else world
            self._check(lib().ts_hydro_set_amr_mesh_partitioned(
                self._h, mesh.n_leaves, _p(nbr, _i64p), _p(lev, _i32p), mesh.max_level, mesh.n_proxy,
                _p(px, _i32p), len(rf), _p(rf, _i32p), _p(own, _i32p), world, rank), "set_amr_mesh")
        self.mesh = None
        self.amr_mesh = mesh
        self.rank = rank

    def local_counts(self):
        a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        self._check(lib().ts_hydro_local_counts(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)),
                    "local_counts")
        return a.value, b.value, c.value

    def owned_ids(self) -> np.ndarray:
        n = self.local_counts()[0]
        out = np.zeros(n, np.int64)
        self._check(lib().ts_hydro_owned_ids(self._h, _p(out, _i64p)), "owned_ids")
        return out

    def halo_plan(self, peer: int):
        ns, nr = ctypes.c_int64(), ctypes.c_int64()
        self._check(lib().ts_hydro_halo_plan(self._h, peer, ctypes.byref(ns), None, ctypes.byref(nr), None), "plan")
        s = np.zeros((max(ns.value, 1), 2), np.int64)
        r = np.zeros((max(nr.value, 1), 2), np.int64)
        self._check(lib().ts_hydro_halo_plan(self._h, peer, ctypes.byref(ns), _p(s, _i64p), ctypes.byref(nr),
                                             _p(r, _i64p)), "plan")
        return s[:ns.value], r[:nr.value]

    def upload(self, U: np.ndarray, first: int = 0) -> None:
        U = np.ascontiguousarray(U, np.float64)
        self._check(lib().ts_hydro_upload(self._h, first, U.shape[0], _p(U, _f64p)), "upload")

    def download(self, first: int = 0, count: Optional[int] = None) -> np.ndarray:
        if count is None:
            count = self.local_counts()[0] - first
        out = np.zeros((count, self.nf, NC), np.float64)
        self._check(lib().ts_hydro_download(self._h, first, count, _p(out, _f64p)), "download")
        return out

    def download_buffer(self, which: int, first: int = 0, count: Optional[int] = None) -> np.ndarray:
        """Diagnostic: RK buffer 0 (U^n), 1 (U^(1)) or 2 (U^(2)), owned + proxy range."""
        if count is None:
            count = self.local_counts()[0] - first
        out = np.zeros((count, self.nf, NC), np.float64)
        self._check(lib().ts_hydro_download_buffer(self._h, which, first, count, _p(out, _f64p)), "download_buffer")
        return out

    def init_random(self, seed: int = 2210) -> None:
        self._check(lib().ts_hydro_init_random(self._h, seed), "init_random")

    # -- persisted state (ts_hydro_ckpt.cpp)
    def save(self, path: str) -> None:
        """U^n of the owned sub-grids + the global mesh -> one checkpoint file."""
        self._check(lib().ts_hydro_save(self._h, os.fsencode(path)), "save")

    def restore(self, paths) -> None:
        """U^n of the owned sub-grids from a checkpoint's files (any writer rank count)."""
        paths = [paths] if isinstance(paths, (str, os.PathLike)) else list(paths)
        arr = (ctypes.c_char_p * len(paths))(*[os.fsencode(p) for p in paths])
        self._check(lib().ts_hydro_restore(self._h, arr, len(paths)), "restore")

    def mesh(self) -> "Mesh":
        """The bound global mesh (Mesh without positions)."""
        n, w, r = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32()
        self._check(lib().ts_hydro_get_mesh(self._h, ctypes.byref(n), None, None, ctypes.byref(w), ctypes.byref(r)),
                    "get_mesh")
        nbr = np.zeros((n.value, 6), np.int64)
        own = np.zeros(n.value, np.int32)
        self._check(lib().ts_hydro_get_mesh(self._h, None, _p(nbr, _i64p), _p(own, _i32p), None, None), "get_mesh")
        return Mesh(nbr, np.zeros((n.value, 3), np.int32), own, w.value)

    # -- stepping
    def compute_dt(self) -> float:
        dt = ctypes.c_double()
        self._check(lib().ts_hydro_compute_dt(self._h, ctypes.byref(dt)), "compute_dt")
        return dt.value

    def step(self, nsteps: int = 1) -> None:
        self._check(lib().ts_hydro_step(self._h, nsteps), "step")

    def step_host(self, host_in: int, host_out: int, nsteps: int = 1) -> None:
        self._check(lib().ts_hydro_step_host(self._h, host_in, host_out, nsteps), "step_host")

    def step_host_async(self, host_in: int, host_out: int, nsteps: int = 1, done=None) -> None:
        """Pipelined step_host (ts_hydro_step_host_async); synchronize() or `done` before reading host_out."""
        self._check(lib().ts_hydro_step_host_async(self._h, host_in, host_out, nsteps, self._done(done), None),
                    "step_host_async")

    def time_steps(self, nsteps: int) -> float:
        """nsteps steps bracketed by CUDA events on the compute stream; device ms."""
        ms = ctypes.c_double()
        self._check(lib().ts_hydro_time_steps(self._h, nsteps, ctypes.byref(ms)), "time_steps")
        return ms.value

    def synchronize(self) -> None:
        self._check(lib().ts_hydro_synchronize(self._h), "synchronize")

    def last_dt(self) -> float:
        dt = ctypes.c_double()
        self._check(lib().ts_hydro_last_dt(self._h, ctypes.byref(dt)), "last_dt")
        return dt.value

    def steps_done(self) -> int:
        v = ctypes.c_uint64()
        self._check(lib().ts_hydro_steps_done(self._h, ctypes.byref(v)), "steps_done")
        return v.value

    def launch_count(self) -> int:
        v = ctypes.c_uint64()
        self._check(lib().ts_hydro_launch_count(self._h, ctypes.byref(v)), "launch_count")
        return v.value

    def launch_stage(self, stage: int, owned_index: Sequence[int], stream_id: int = 0, guid: int = 0,
                     done=None) -> None:
        """The compute_fluxes drop-in (workload.cpp:544-552); `done()` fires after the device finished."""
        idx = np.ascontiguousarray(np.asarray(owned_index, np.int64))
        cb = DONE_FN(lambda _u: done()) if done is not None else DONE_FN()
        if done is not None:
            self._callbacks.append(cb)
        self._check(lib().ts_hydro_launch_stage(self._h, stage, _p(idx, _i64p), len(idx), stream_id, guid, cb, None),
                    "launch_stage")

    def gravity_p2p(self, G: float = 1.0, radius: int = 4, owned_index=None, stream_id: int = 0, guid: int = 0,
                    done=None) -> None:
        """Near-field monopole P2P (the reference's p2p_kernel launches, workload.cpp:365-372)."""
        if owned_index is None:
            idx, n = None, 0
        else:
            idx = np.ascontiguousarray(np.asarray(owned_index, np.int64))
            n = len(idx)
        self._check(lib().ts_hydro_gravity_p2p(self._h, G, radius, None if idx is None else _p(idx, _i64p), n,
                                               stream_id, guid, self._done(done), None), "gravity_p2p")

    def gravity_tree_of_mesh(self):
        """(level, pos, dims, dx0) of the bound mesh's leaves, for set_gravity_tree."""
        if getattr(self, "amr_mesh", None) is not None and getattr(self, "mesh", None) is None:
            m = self.amr_mesh
            return m.level, m.pos, m.dims, self.config.dx * 2.0 ** m.max_level
        m = self.mesh
        return np.zeros(m.n, np.int32), m.pos, m.dims, self.config.dx

    def set_gravity_tree(self, level=None, pos=None, dims=None, dx0: Optional[float] = None) -> None:
        """Bind the octree of the owned sub-grids for gravity_fmm (default: the bound mesh's own)."""
        if level is None:
            level, pos, dims, dx0 = self.gravity_tree_of_mesh()
        lev = np.ascontiguousarray(level, np.int32)
        ps = np.ascontiguousarray(np.asarray(pos).reshape(-1, 3), np.int32)
        dm = np.ascontiguousarray(dims, np.int32)
        self._check(lib().ts_hydro_set_gravity_tree(self._h, len(lev), _p(lev, _i32p), _p(ps, _i32p), _p(dm, _i32p),
                                                    float(dx0)), "set_gravity_tree")

    def gravity_fmm(self, G: float = 1.0, radius: int = 2, stream_id: int = 0, guid: int = 0, done=None) -> None:
        """Whole gravity solve (FMM over the octree; the reference's multipole_root / multipole /
        p2m / p2p launches, workload.cpp:365-372).  Result: download_gravity()."""
        self._check(lib().ts_hydro_gravity_fmm(self._h, G, radius, stream_id, guid, self._done(done), None),
                    "gravity_fmm")

    def gravity_kick(self, dt: float = -1.0) -> None:
        """Gravity source over dt from the last solve (dt < 0: the last step's dt)."""
        self._check(lib().ts_hydro_gravity_kick(self._h, dt), "gravity_kick")

    def step_gravity(self, nsteps: int = 1, G: float = 1.0, radius: int = 2) -> None:
        """nsteps of hydro + self-gravity (step, FMM, kick), all on the device."""
        self._check(lib().ts_hydro_step_gravity(self._h, nsteps, G, radius), "step_gravity")

    def download_gravity(self, first: int = 0, count: Optional[int] = None) -> np.ndarray:
        n = self.local_counts()[0] if count is None else count
        out = np.zeros((n, 4, N * N * N), np.float64)
        self._check(lib().ts_hydro_download_gravity(self._h, first, n, _p(out, _f64p)), "download_gravity")
        return out

    def finish_step(self) -> None:
        self._check(lib().ts_hydro_finish_step(self._h), "finish_step")

    # -- ghost exchange
    def exchange_faces(self) -> np.ndarray:
        n = self.local_counts()[0]
        out = np.zeros((n, 6, N * N), np.float64)
        self._check(lib().ts_hydro_exchange_faces(self._h, _p(out, _f64p)), "exchange_faces")
        return out

    def fill_halo(self, depth: int = 3) -> np.ndarray:
        n = self.local_counts()[0]
        pe = N + 2 * depth
        out = np.zeros((n, self.nf, pe, pe, pe), np.float64)
        self._check(lib().ts_hydro_fill_halo(self._h, depth, _p(out, _f64p)), "fill_halo")
        return out

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        rc = lib().ts_hydro_nccl_unique_id(buf)
        if rc != TS_OK:
            raise TsError(rc, "ncclGetUniqueId failed")
        return buf.raw

    def comm_init(self, uid: bytes, nranks: int, rank: int) -> None:
        self._check(lib().ts_hydro_comm_init(self._h, uid, nranks, rank), "comm_init")

    def p2p_export(self) -> bytes:
        """This rank's P2P blob (IPC handles + receive offsets) for the all-gather."""
        n = lib().ts_hydro_p2p_blob_size()
        buf = ctypes.create_string_buffer(n)
        self._check(lib().ts_hydro_p2p_export(self._h, buf), "p2p_export")
        return buf.raw

    def p2p_import(self, blobs: Sequence[bytes]) -> None:
        """Open every rank's blob (rank order) and switch the halo/dt transport to P2P."""
        data = b"".join(blobs)
        self._check(lib().ts_hydro_p2p_import(self._h, data, len(blobs)), "p2p_import")

    def selftest_math(self, n: int, seed: int = 1, emax: int = 1000):
        """(rcp mismatches, sqrt mismatches) of the branch-free EOS math vs IEEE on n samples."""
        a, b = ctypes.c_uint64(), ctypes.c_uint64()
        self._check(lib().ts_hydro_selftest_math(self._h, n, seed, emax, ctypes.byref(a), ctypes.byref(b)),
                    "selftest_math")
        return a.value, b.value

    def halo_exchange(self) -> None:
        self._check(lib().ts_hydro_halo_exchange(self._h), "halo_exchange")

    # -- timing hook
    def flush_activity(self) -> list:
        n = ctypes.c_uint64()
        self._check(lib().ts_hydro_flush_activity(self._h, None, 0, ctypes.byref(n)), "flush_activity")
        buf = (_Record * max(n.value, 1))()
        self._check(lib().ts_hydro_flush_activity(self._h, buf, n.value, ctypes.byref(n)), "flush_activity")
        return [ActivityRecord(ACTIVITY_KINDS[r.kind], r.name.decode(), r.device_id, r.stream_id, r.start_ns,
                               r.end_ns, r.bytes if r.has_bytes else None, r.correlation_guid)
                for r in buf[:n.value]]

    def debug_check(self, reset: bool = False):
        """Self-check build counters: (failures, first code, a, b, code bitmask) — DESIGN.md §13."""
        out = np.zeros(5, np.uint64)
        self._check(lib().ts_hydro_debug_check(self._h, _p(out, _u64p), 1 if reset else 0), "debug_check")
        return tuple(int(x) for x in out)

    def set_profiling(self, enabled: bool) -> None:
        """ProfilingArm full (True) / disabled (False): activity stamps and records on or off."""
        self._check(lib().ts_hydro_set_profiling(self._h, 1 if enabled else 0), "set_profiling")

    def set_activity_sink(self, fn) -> None:
        def thunk(recs, n, _u):
            fn([ActivityRecord(ACTIVITY_KINDS[recs[i].kind], recs[i].name.decode(), recs[i].device_id,
                               recs[i].stream_id, recs[i].start_ns, recs[i].end_ns,
                               recs[i].bytes if recs[i].has_bytes else None, recs[i].correlation_guid)
                for i in range(n)])
        self._sink = SINK_FN(thunk) if fn is not None else SINK_FN()
        self._check(lib().ts_hydro_set_activity_sink(self._h, self._sink, None), "set_activity_sink")

    def memory_state(self) -> dict:
        m = _MemState()
        self._check(lib().ts_hydro_memory_state(self._h, ctypes.byref(m)), "memory_state")
        return {k: getattr(m, k) for k, _ in m._fields_}

    def host_pinned_alloc(self, nbytes: int) -> int:
        p = _vp()
        self._check(lib().ts_hydro_host_alloc(self._h, nbytes, ctypes.byref(p)), "host_pinned_alloc")
        return p.value

    def host_pinned_free(self, ptr: int) -> None:
        self._check(lib().ts_hydro_host_free(self._h, ptr), "host_pinned_free")

    # -- the rest of the SimDevice contract (device.hpp:57-64) on the GPU
    def _done(self, done):
        cb = DONE_FN(lambda _u: done()) if done is not None else DONE_FN()
        if done is not None:
            self._callbacks.append(cb)
        return cb

    def launch_kernel(self, name: str, stream_id: int, duration_ns: int, guid: int = 0, done=None) -> None:
        """SimDevice::launch_kernel: `name` occupies `stream_id` for duration_ns on the GPU."""
        self._check(lib().ts_hydro_launch_kernel(self._h, name.encode(), stream_id, duration_ns, guid,
                                                 self._done(done), None), "launch_kernel")

    def enqueue_copy(self, kind: str, nbytes: int, stream_id: int, guid: int = 0, done=None) -> None:
        """SimDevice::enqueue_copy: a real copy of nbytes ("copy_host_to_device", ...)."""
        k = ACTIVITY_KINDS.index(kind) if kind in ACTIVITY_KINDS else -1
        self._check(lib().ts_hydro_enqueue_copy(self._h, k, nbytes, stream_id, guid, self._done(done), None),
                    "enqueue_copy")

    def device_alloc(self, nbytes: int) -> int:
        h = ctypes.c_uint64()
        self._check(lib().ts_hydro_device_alloc(self._h, nbytes, ctypes.byref(h)), "device_alloc")
        return h.value

    def device_free(self, handle: int) -> None:
        self._check(lib().ts_hydro_device_free(self._h, handle), "device_free")

    def debug_cta_log(self) -> np.ndarray:
        """[3][n_owned][4] per-CTA {SM, start, work start, end} of the last step (TS_HYDRO_CTA_LOG)."""
        n = ctypes.c_uint64()
        self._check(lib().ts_hydro_debug_cta_log(self._h, None, 0, ctypes.byref(n)), "debug_cta_log")
        out = np.zeros(max(n.value, 1), np.uint64)
        self._check(lib().ts_hydro_debug_cta_log(self._h, _p(out, _u64p), out.size, ctypes.byref(n)), "debug_cta_log")
        return out[:n.value].reshape(3, -1, 4) if n.value else out[:0].reshape(3, 0, 4)

    def device_ptr(self, handle: int) -> int:
        p = _vp()
        if lib().ts_hydro_device_ptr(self._h, handle, ctypes.byref(p)) != TS_OK:
            raise ValueError("unknown device handle")
        return p.value


def clock_ns() -> int:
    return lib().ts_hydro_clock_ns()


# ---------------------------------------------------------------------------
# Session (WorkloadSession, workload.hpp:165-214)
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class ScalingPoint:
    """workload.hpp:129-137."""
    n: int = 1
    total_time_s: float = 0.0
    cells_per_second: float = 0.0
    speedup: float = 1.0


class WorkloadSession:
    """Binds a mesh to a device and steps it.  Only stepping is timed
    (workload.cpp:595-612); cells/s = total_cells * num_steps / seconds."""

    def __init__(self, mesh: Mesh, device: CudaDevice, config: StepConfig = None, rank: int = 0):
        self.config = config or StepConfig()
        self.config.validate()
        if mesh.world_size > 1 and rank >= mesh.world_size:
            raise ValueError("rank outside the mesh partition")
        self.mesh = mesh
        self.device = device
        self.rank = rank
        device.set_mesh(mesh, rank)

    def load_problem(self, problem: str, seed: int = 2210) -> None:
        if problem == "random_device":
            self.device.init_random(seed)
            return
        ids = self.device.owned_ids()
        self.device.upload(ic_fill(self.device.config, problem, self.mesh, ids, seed))

    def exchange_ghost_cells(self, mode: str = "direct_local", step: int = 0) -> np.ndarray:
        """One reference-shaped face exchange of field 0 (workload.cpp:572-581)."""
        if mode not in ("remote_action", "direct_local"):
            raise ValueError(f"unknown comm mode '{mode}'")
        return self.device.exchange_faces()

    def run_step(self, step_index: int = 0) -> int:
        t0 = time.perf_counter_ns()
        self.device.step(1)
        self.device.synchronize()
        return time.perf_counter_ns() - t0

    def run_benchmark(self) -> ScalingPoint:
        if self.config.num_steps == 0:
            raise ValueError("num_steps must be positive for a benchmark run")
        self.device.synchronize()
        t0 = time.perf_counter()
        self.device.step(self.config.num_steps)
        self.device.synchronize()
        seconds = time.perf_counter() - t0
        return ScalingPoint(n=self.mesh.world_size, total_time_s=seconds,
                            cells_per_second=self.mesh.total_cells() * self.config.num_steps / seconds)


# ---------------------------------------------------------------------------
# Overhead / scaling harness (reference proj/core/src/harness.cpp): the
# profiling-overhead percentage, the sweep rows derived from per-count times,
# and the CSV writer — restated so a sweep over GPU counts produces the
# reference's own row format.  The "with" arm runs the per-kernel timing hook
# (activity stamps), "without" runs with it disabled (ts_hydro_set_profiling).
# ---------------------------------------------------------------------------
def compute_overhead(n: int, comp_apex_s: float, comp_no_apex_s: float) -> float:
    """harness.cpp:15-20: (with / without) * 100 - 100 percent."""
    del n
    if not comp_no_apex_s > 0.0:
        raise ValueError("overhead baseline must be positive")
    return (comp_apex_s / comp_no_apex_s) * 100.0 - 100.0


@dataclasses.dataclass
class SweepRow:
    """harness.hpp:66-75."""
    n: int = 1
    time_with_s: float = 0.0
    time_without_s: float = 0.0
    cells_per_second_with: float = 0.0
    cells_per_second_without: float = 0.0
    o_percent: float = 0.0
    speedup_with: float = 1.0     # relative to the smallest count, same arm
    speedup_without: float = 1.0


def _validate_counts(counts: Sequence[int]) -> None:
    """harness.cpp:125-132."""
    if len(counts) == 0:
        raise ValueError("sweep needs at least one locality count")
    for i, c in enumerate(counts):
        if c < 1:
            raise ValueError("locality counts must be positive")
        if i > 0 and c <= counts[i - 1]:
            raise ValueError("locality counts must be strictly ascending")


def sweep_rows_from_times(total_cells: int, num_steps: int, counts: Sequence[int], with_s: Sequence[float],
                          without_s: Sequence[float]) -> list:
    """harness.cpp:136-167.  cells processed = the world-1 mesh's total cells
    x num_steps (the reference rebuilds build_mesh(levels, 1, ...) for it;
    here the caller passes that mesh's total_cells — for weak scaling the
    per-count mesh differs, and tools/sweep.py passes each row's own)."""
    _validate_counts(counts)
    if len(with_s) != len(counts) or len(without_s) != len(counts):
        raise ValueError("sweep needs one time per arm per locality count")
    for a, b in zip(with_s, without_s):
        if not (a > 0.0) or not (b > 0.0):
            raise ValueError("sweep times must be positive")
    cells_processed = float(total_cells) * float(num_steps)
    rows = []
    for i, n in enumerate(counts):
        rows.append(SweepRow(n=n, time_with_s=with_s[i], time_without_s=without_s[i],
                             cells_per_second_with=cells_processed / with_s[i],
                             cells_per_second_without=cells_processed / without_s[i],
                             o_percent=compute_overhead(n, with_s[i], without_s[i]),
                             speedup_with=with_s[0] / with_s[i], speedup_without=without_s[0] / without_s[i]))
    return rows


def write_sweep_csv(out, rows) -> None:
    """harness.cpp:188-201: fixed header, doubles as %.17g (exact round trip)."""
    out.write("n,time_with,time_without,cells_per_second_with,cells_per_second_without,"
              "o_percent,speedup_with,speedup_without\n")
    for r in rows:
        vals = (r.time_with_s, r.time_without_s, r.cells_per_second_with, r.cells_per_second_without,
                r.o_percent, r.speedup_with, r.speedup_without)
        out.write(str(r.n) + "".join("," + ("%.17g" % v) for v in vals) + "\n")


def measure_arm(session: "WorkloadSession", profiling: bool, repetitions: int = 3) -> float:
    """harness.cpp:72-101 on the GPU: min over repetitions of the timed
    stepping (run_benchmark) with the timing hook on (full) or off (disabled)."""
    if repetitions < 1:
        raise ValueError("repetitions must be positive")
    session.device.set_profiling(profiling)
    try:
        best = float("inf")
        for _ in range(repetitions):
            best = min(best, session.run_benchmark().total_time_s)
    finally:
        session.device.set_profiling(True)
    session.device.flush_activity()
    return best


# ---------------------------------------------------------------------------
# Checkpoint files (host side, no GPU): ts_hydro_checkpoint_{write,info,read}
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class Checkpoint:
    """One checkpoint file: header fields, the global mesh, and the stored
    sub-grids' U^n ([n_records][nf][512], in global_ids order)."""
    header: dict
    neighbor_ids: np.ndarray
    owner: np.ndarray
    global_ids: np.ndarray
    state: np.ndarray


def write_checkpoint(path: str, cfg: HydroConfig, mesh: Mesh, global_ids, state, steps_done: int = 0,
                     rank: int = 0) -> None:
    gids = np.ascontiguousarray(global_ids, np.int64)
    st = np.ascontiguousarray(state, np.float64)
    if st.shape != (gids.size, cfg.nf, NC):
        raise ValueError(f"state shape {st.shape} != ({gids.size}, {cfg.nf}, {NC})")
    nbr = np.ascontiguousarray(mesh.neighbor_ids, np.int64)
    own = np.ascontiguousarray(mesh.owner, np.int32)
    c = cfg.to_c()
    rc = lib().ts_hydro_checkpoint_write(os.fsencode(path), ctypes.byref(c), mesh.n, _p(nbr, _i64p), _p(own, _i32p),
                                         mesh.world_size, rank, gids.size, _p(gids, _i64p), _p(st, _f64p),
                                         steps_done)
    if rc != TS_OK:
        raise ValueError(f"cannot write checkpoint {path}")


def read_checkpoint(path: str) -> Checkpoint:
    """Validated read (magic, version, sizes, payload checksum); ValueError otherwise."""
    h = _CkptHeader()
    if lib().ts_hydro_checkpoint_info(os.fsencode(path), ctypes.byref(h)) != TS_OK:
        raise ValueError(f"checkpoint {path}: unreadable, truncated or corrupt")
    nbr = np.zeros((h.n_grids, 6), np.int64)
    own = np.zeros(h.n_grids, np.int32)
    gid = np.zeros(h.n_records, np.int64)
    st = np.zeros((h.n_records, h.nf, NC), np.float64)
    if lib().ts_hydro_checkpoint_read(os.fsencode(path), _p(nbr, _i64p), _p(own, _i32p), _p(gid, _i64p),
                                      _p(st, _f64p)) != TS_OK:
        raise ValueError(f"checkpoint {path}: read failed")
    hdr = {k: getattr(h, k) for k, _ in _CkptHeader._fields_}
    return Checkpoint(hdr, nbr, own, gid, st)
