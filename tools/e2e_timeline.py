"""Timeline of the pipelined host-buffer steps (ts_hydro_step_host_async):
per step, when the H2D, the stages and the D2H ran (activity records)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2210_06437_b200 import hydro as H  # noqa: E402

m = H.uniform_mesh(16, 16, 16)
cfg = H.HydroConfig(dx=1.0 / 128)
dev = H.CudaDevice(cfg)
dev.set_mesh(m)
dev.upload(H.ic_fill(cfg, "sedov", m, range(m.n)))
U = dev.download()
hin, hout = dev.host_pinned_alloc(U.nbytes), dev.host_pinned_alloc(U.nbytes)
ctypes.memmove(hin, U.ctypes.data, U.nbytes)
for _ in range(3):
    dev.step_host_async(hin, hout, 1)
    hin, hout = hout, hin
dev.synchronize()
dev.flush_activity()
for _ in range(4):
    dev.step_host_async(hin, hout, 1)
    hin, hout = hout, hin
dev.synchronize()
recs = sorted(dev.flush_activity(), key=lambda r: r.start_ns)
t0 = recs[0].start_ns
for r in recs:
    print(f"{r.name:24s} s{r.stream_id:<3d} {(r.start_ns - t0) / 1e3:9.1f} -> {(r.end_ns - t0) / 1e3:9.1f} us"
          f"  ({(r.end_ns - r.start_ns) / 1e3:7.1f})")
