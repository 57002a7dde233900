"""PCIe ceiling of the e2e path: pinned H2D alone, D2H alone, and both at once
on two streams (100 MB each, like one Sedov step's state)."""
import json
import time

import torch

n = 100 * 1024 * 1024 // 8
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                d_a.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_out.copy_(d_b, non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


run(True, True, 2)
t_h, t_d, t_b = run(True, False), run(False, True), run(True, True)
mb = n * 8 / 1e9
print(json.dumps({"h2d_GBps": mb / t_h, "d2h_GBps": mb / t_d, "both_GBps_each": mb / t_b,
                  "both_ms_per_100MB_pair": t_b * 1e3,
                  "e2e_ceiling_Gcells": 2097152 / t_b / 1e9}))
