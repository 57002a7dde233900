#!/bin/bash
# DRAM bytes per stage launch (ncu, cold-cache replays) for Morton vs row numbering, nf 6 and nf 11.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/traffic
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for w in sedov polytrope; do
for o in morton row; do
  timeout 900 ncu --metrics $M --clock-control none -k regex:stage_kernel --launch-skip 12 --launch-count 3 --csv \
    python bench.py --workload $w --order $o --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/traffic/${w}_${o}.csv 2>&1
  echo "$w $o rc=$?"
done
done
python - <<'PY'
import csv, glob
alg = {"sedov": (6, 4096), "polytrope": (11, 32768)}
for f in sorted(glob.glob("gpurun_out/traffic/*.csv")):
    w, o = f.split("/")[-1][:-4].split("_")
    rows = [x for x in csv.reader(open(f)) if len(x) > 14 and x[0].isdigit()]
    d = {}
    for x in rows:
        d.setdefault(x[0], {})[x[12]] = float(x[14])
    nf, n = alg[w]
    tot = sum(v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"] for v in d.values())
    t = sum(v["gpu__time_duration.sum"] for v in d.values())
    a = 64 * nf * n * 512  # algorithmic bytes of one step = 3 stage launches
    print(f"{w:10s} {o:7s} DRAM {tot/1e9:7.3f} GB per step vs algorithmic {a/1e9:7.3f} GB: {tot/a:5.3f}x   stage time {t/1e3:8.1f} us")
PY
