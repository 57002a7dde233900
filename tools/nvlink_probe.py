"""Probe the NVLink counters NVML exposes on this box (2-GPU gpurun call)."""
import subprocess

import pynvml

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
names = [n for n in dir(pynvml) if n.startswith("NVML_FI_DEV_NVLINK") and ("THROUGHPUT" in n or "COUNT_XMIT" in n
                                                                             or "COUNT_RCV" in n or "BYTES" in n)]
for n in names:
    fid = getattr(pynvml, n)
    for scope in (0, 1, 0xFFFFFFFF):
        try:
            r = pynvml.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            print(n, fid, hex(scope), "ret", r.nvmlReturn, "val", r.value.ullVal)
        except Exception as e:
            print(n, fid, hex(scope), "exc", e)
for link in range(18):
    try:
        st = pynvml.nvmlDeviceGetNvLinkState(h, link)
        print("link", link, "state", st)
    except Exception as e:
        print("link", link, "exc", e)
        break
print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout)
print(subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", "0"], capture_output=True, text=True).stdout[:3000])
