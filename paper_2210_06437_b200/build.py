"""Build recipe for libts_hydro.so (sm_100a), in-tree.

    python -m paper_2210_06437_b200.build [--force] [-j N]

Every .cu is compiled by nvcc for ``-gencode arch=compute_100a,code=sm_100a``
with ``--fmad=false`` (no implicit contraction: the numerics contract names
every fma) and ``-lineinfo`` (ncu source view); host C++ by g++; all linked
into ``paper_2210_06437_b200/libts_hydro.so`` with the static CUDA runtime.
The per-field-count stage kernels live in separate translation units so they
compile in parallel.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(os.path.dirname(PKG), "include")
# Tuning builds: TS_VARIANT=name TS_DEFINES="-DTS_MINB=8" -> build_name/ + libts_hydro_name.so
VARIANT = os.environ.get("TS_VARIANT", "")
BUILD = os.path.join(PKG, "build" + (f"_{VARIANT}" if VARIANT else ""))
LIB = os.path.join(PKG, "libts_hydro" + (f"_{VARIANT}" if VARIANT else "") + ".so")
EXTRA = os.environ.get("TS_DEFINES", "").split()
NVCC_EXTRA = os.environ.get("TS_NVCC_FLAGS", "").split()  # nvcc only (e.g. -Xptxas options)

CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = shutil.which("nvcc") or os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-Xptxas", "-warn-spills", f"-I{INCLUDE}", f"-I{CSRC}"]
CXX_FLAGS = ["-O2", "-fPIC", "-std=c++17", "-ffp-contract=off", "-Wall", "-Wextra", f"-I{INCLUDE}",
             f"-I{CSRC}", f"-I{CUDA_HOME}/include"]


def _headers():
    return glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(INCLUDE, "*.h"))


def _stale(obj: str, src: str, deps) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(p) > t for p in [src, *deps])


def _compile(src: str, force: bool):
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    if not force and not _stale(obj, src, _headers()):
        return obj, None
    if src.endswith(".cu"):
        cmd = [NVCC, *NVCC_FLAGS, *EXTRA, *NVCC_EXTRA, "-c", src, "-o", obj]
    else:
        cmd = ["g++", *CXX_FLAGS, *EXTRA, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return obj, (r.stdout + r.stderr).strip()


def build(force: bool = False, jobs: int | None = None, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    jobs = jobs or max(1, os.cpu_count() or 1)
    with cf.ThreadPoolExecutor(jobs) as ex:
        results = list(ex.map(lambda s: _compile(s, force), srcs))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log:
                print(log)
    if force or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-ldl", "-lpthread", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if not VARIANT:
        _build_driver(force)
    return LIB


DRIVER_SRC = os.path.join(os.path.dirname(PKG), "tools", "ts_hydro_run.cpp")
DRIVER = os.path.join(os.path.dirname(PKG), "tools", "ts_hydro_run")


def _build_driver(force: bool) -> None:
    """The native C++ host driver over the C ABI (tools/ts_hydro_run.cpp)."""
    if not os.path.exists(DRIVER_SRC):
        return
    if not force and os.path.exists(DRIVER) and os.path.getmtime(DRIVER) >= max(
            os.path.getmtime(DRIVER_SRC), os.path.getmtime(LIB)):
        return
    cmd = ["g++", "-O2", "-std=c++17", "-Wall", f"-I{INCLUDE}", DRIVER_SRC, f"-L{PKG}", "-l:libts_hydro.so",
           f"-Wl,-rpath,{PKG}", "-o", DRIVER]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"driver build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    ap.add_argument("-v", action="store_true")
    a = ap.parse_args(argv)
    print(build(a.force, a.j, a.v))
    return 0


if __name__ == "__main__":
    sys.exit(main())
