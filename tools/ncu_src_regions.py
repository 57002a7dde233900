"""Split an ncu source-page CSV (--page source --print-source=sass) of one
kernel into loop regions (backward branches) and print the warp-stall samples
per region and reason: where the stage kernel spends its time."""
import csv
import re
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    data = []
    for r in rows[2:]:
        if r and r[0] == "Kernel Name":
            break  # the next kernel's block
        data.append(r)
    ia, isrc, isamp = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    iexec = hdr.index("Instructions Executed")
    stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_")]
    addr = [int(r[ia], 16) for r in data]
    base = addr[0]
    loops = []
    for k, r in enumerate(data):
        m = re.search(r"BRA(?:\.\w+)*\s+(?:!?U?P\w+,\s*)?(0x[0-9a-f]+)", r[isrc])
        if m:
            tgt = int(m.group(1), 16) - base
            if tgt < addr[k] - base:  # backward: a loop
                loops.append((tgt, addr[k] - base))
    loops.sort()
    tot = sum(float(r[isamp] or 0) for r in data)
    print(f"total samples {tot:.0f}")
    for lo, hi in loops:
        sel = [r for r, a in zip(data, addr) if lo <= a - base <= hi]
        s = sum(float(r[isamp] or 0) for r in sel)
        if s < 0.01 * tot:
            continue
        ex = max(int(r[iexec] or 0) for r in sel)
        st = defaultdict(float)
        for r in sel:
            for i, h in stall_cols:
                st[h] += float(r[i] or 0)
        top = sorted(st.items(), key=lambda kv: -kv[1])[:7]
        ninstr = len(sel)
        print(f"loop 0x{lo:x}-0x{hi:x} ({ninstr} instr, max exec {ex}): {100 * s / tot:5.1f}% of samples; "
              + ", ".join(f"{h[6:]} {100 * v / s:.0f}%" for h, v in top))


if __name__ == "__main__":
    main(sys.argv[1])
