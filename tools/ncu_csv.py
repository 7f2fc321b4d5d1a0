"""Print an `ncu --metrics ... --csv` launch list (stdout of the profiled command may precede it)."""
import csv
import sys
from collections import defaultdict


def load(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    hdr = rows[0]
    ki, mi, vi, ii = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    d = defaultdict(dict)
    for r in rows[1:]:
        if len(r) == len(hdr):
            d[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
            d[int(r[ii])]["kernel"] = r[ki].split("(")[0].replace("void ", "").replace("mlora::", "")
    return [d[i] for i in sorted(d)]


if __name__ == "__main__":
    for path in sys.argv[1:]:
        print(path)
        rows = load(path)
        keys = [k for k in rows[0] if k != "kernel"]
        print("  kernel | " + " | ".join(keys))
        for r in rows:
            print("  " + r["kernel"][:32] + " | " + " | ".join(f"{r[k]:.4g}" for k in keys))
