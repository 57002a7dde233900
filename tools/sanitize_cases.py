"""Small GPU cases for compute-sanitizer (memcheck / synccheck / racecheck /
initcheck): every hand-rolled synchronisation protocol of the path runs once
on a mesh small enough for the instrumented run, each checked against the
oracle or the stream-ordered run.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2210_06437_b200 import hydro as H  # noqa: E402


CHECKED = []


def ok(name, cond, dev=None):
    """Parity against the oracle, plus (TS_CHECK library) the device's
    self-check counters: bounds of every state access, every acquired flag
    still at its awaited value at CTA exit."""
    chk = ""
    if dev is not None and H.lib().ts_hydro_check_build():
        n, code, a, b, _ = dev.debug_check(reset=True)
        CHECKED.append(n)
        chk = f"  [self-check: {n} failures" + (f", first code {code} ({a}, {b})" if n else "") + "]"
        cond = cond and n == 0
    print(("OK   " if cond else "FAIL ") + name + chk, flush=True)
    if not cond:
        sys.exit(1)


def main():
    p6 = oracle.params(nf=6, dx=1.0 / 64)
    # 1. batched steps with the single-rank dataflow (PDL dependents, per-sub-grid flags,
    #    stage-3 count -> next stage 1) vs the oracle
    m = H.uniform_mesh(8, 8, 8)
    U0 = oracle.ic_sedov(p6, m.pos, (8, 8, 8))
    d = H.CudaDevice(H.HydroConfig(dx=1.0 / 64))
    d.set_mesh(m)
    d.upload(U0)
    d.step(3)
    d.synchronize()
    want, _ = oracle.run(p6, m.neighbor_ids, U0, 3, nthreads=os.cpu_count() or 1)
    ok("dataflow steps (PDL + flow flags + stage-3 count)", np.array_equal(d.download(), want), d)
    # 2. per-sub-grid drop-in: device-side flags across 16 streams, no host barrier
    d.upload(U0)
    d.compute_dt()
    for _ in range(2):
        for stage in (1, 2, 3):
            for g in range(m.n):
                d.launch_stage(stage, [g], stream_id=(g * 7 + stage) % 16)
        d.finish_step()
    d.synchronize()
    want2, _ = oracle.run(p6, m.neighbor_ids, U0, 2, nthreads=os.cpu_count() or 1)
    ok("drop-in launches (flags, inline lists, lead CTA)", np.array_equal(d.download(), want2), d)
    # 3. pipelined host steps: chained calls (H2D chunk flags gate stage 1,
    #    stage-3 chunk counters gate the D2H)
    nbytes = U0.nbytes
    hin, hout = d.host_pinned_alloc(nbytes), d.host_pinned_alloc(nbytes)
    ctypes.memmove(hin, U0.ctypes.data, nbytes)
    for _ in range(3):
        d.step_host_async(hin, hout, 1)
        hin, hout = hout, hin
    d.synchronize()
    got = np.empty_like(U0)
    ctypes.memmove(got.ctypes.data, hin, nbytes)
    ok("pipelined host steps (H2D flags, chunk counters)", np.array_equal(got, want), d)
    d.host_pinned_free(hin)
    d.host_pinned_free(hout)
    d.close()
    # 4. coarse-fine AMR (proxy fill + fused multi-level stage + reflux)
    from paper_2210_06437_b200 import amr
    mesh = amr.amr_mesh(4, 4, 4, {(0, 1, 1, 1), (0, 2, 1, 1), (0, 1, 2, 1), (0, 1, 1, 2), (0, 2, 2, 2)})
    Ua = amr.ic_blast(mesh, 6, 1.0 / 64, width=0.06, centre=(0.625, 0.625, 0.5), drift=(0.3, -0.1, 0.2))
    wa, _ = oracle.run_amr(oracle.params(nf=6, dx=1.0 / 64), mesh, Ua, 2)
    da = H.CudaDevice(H.HydroConfig(dx=1.0 / 64))
    da.set_amr_mesh(mesh)
    da.upload(Ua[:mesh.n_leaves])
    da.step(2)
    da.synchronize()
    ok("AMR steps (fill, level-tagged stage, reflux)", np.array_equal(da.download(), wa[:mesh.n_leaves]), da)
    da.close()
    # 5. the detector itself: a deliberately broken ordering (stages 2, 3 wait
    #    for the previous step's flags) must be reported
    if H.lib().ts_hydro_check_build():
        os.environ["TS_HYDRO_DEBUG_BREAK_FLOW"] = "1"
        db = H.CudaDevice(H.HydroConfig(dx=1.0 / 64))
        db.set_mesh(m)
        db.upload(U0)
        db.step(3)
        db.synchronize()
        n, code, a, b, seen = db.debug_check(reset=True)
        del os.environ["TS_HYDRO_DEBUG_BREAK_FLOW"]
        db.close()
        codes = [k for k in range(64) if (seen >> k) & 1]
        hit = n > 0 and 10 in codes
        print(("OK   " if hit else "FAIL ") +
              f"broken ordering detected: {n} failures, codes {codes} (10 = a flag overtaken, 20 = non-finite "
              f"output); first code {code} ({a}, {b})", flush=True)
        if not hit:
            sys.exit(1)
    print("SANITIZE CASES DONE" + (f" (self-check build, {len(CHECKED)} devices checked)" if CHECKED else ""), flush=True)


if __name__ == "__main__":
    main()
