"""Executed-instruction mix of one kernel from an .ncu-rep source page (SASS)."""
import collections
import csv
import io
import subprocess
import sys


def main(path, idx=0, top=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks, cur = [], None
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "Kernel Name":
            cur = [r]
            blocks.append(cur)
        elif cur is not None:
            cur.append(r)
    b = blocks[int(idx)]
    print(b[0][1])
    hdr = b[1]
    isrc, iex = hdr.index("Source"), hdr.index("Instructions Executed")
    cnt = collections.Counter()
    total = 0
    for r in b[2:]:
        try:
            n = float(r[iex] or 0)
        except ValueError:
            continue
        op = r[isrc].strip()
        if op.startswith("@"):
            op = op.split(None, 1)[1]
        op = op.split()[0].split(".")[0] if op else "?"
        cnt[op] += n
        total += n
    print(f"total warp-instructions {total:.4g}")
    for op, n in cnt.most_common(int(top)):
        print(f"  {op:10s} {n:12.4g}  {100 * n / total:5.1f}%")


if __name__ == "__main__":
    main(*sys.argv[1:])
