"""Print the bench lines of gpurun_out/variants.log compactly."""
import json
import sys

cur = None
for line in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/variants.log"):
    if line.startswith("=="):
        cur = line.strip()
        continue
    if line.startswith("{"):
        d = json.loads(line)
        r = d["roofline"]
        print(f"{cur:60s} {d['value'] / 1e9:7.3f} G/s  frac={r['frac']:.3f}  ms/step={d['ms_per_step']:.3f}")
    elif "Error" in line or "error" in line:
        print(cur, line.strip()[:200])
