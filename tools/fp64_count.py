"""FP64-pipe instruction count per cell-update from an ncu report (source page,
SASS thread-instructions executed) of the three stage kernels."""
import csv
import io
import subprocess
import sys

FP64 = {"DADD", "DMUL", "DFMA", "DSETP"}


def per_cell_update(path, cells):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks, cur = [], None
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "Kernel Name":
            cur = [r]
            blocks.append(cur)
        elif cur is not None:
            cur.append(r)
    total = 0.0
    for b in blocks[:3]:
        hdr = b[1]
        isrc, iex = hdr.index("Source"), hdr.index("Thread Instructions Executed")
        for r in b[2:]:
            op = r[isrc].strip()
            if op.startswith("@"):
                op = op.split(None, 1)[1]
            if op and op.split()[0].split(".")[0] in FP64:
                try:
                    total += float(r[iex] or 0)
                except ValueError:
                    pass
    return total / cells, len(blocks[:3])


if __name__ == "__main__":
    v, n = per_cell_update(sys.argv[1], float(sys.argv[2]))
    print(f"{v:.0f} FP64 thread-instructions per cell-update over {n} stage kernels")
