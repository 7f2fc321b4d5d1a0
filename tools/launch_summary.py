"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel.

    python tools/launch_summary.py launches.csv [steps]
"""
import collections
import csv
import re
import sys


def main():
    path = sys.argv[1]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    H, data = rows[hdr], rows[hdr + 1:]
    ki, vi, ui = H.index("Kernel Name"), H.index("Metric Value"), H.index("Metric Unit")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in data:
        name = re.split(r"[(]", r[ki].replace("(anonymous namespace)::", "").replace("<unnamed>::", ""))[0]
        name = name.replace("void ", "").strip()
        scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}[r[ui]]
        tot[name] += float(r[vi].replace(",", "")) * scale
        cnt[name] += 1
    T = sum(tot.values())
    print(f"{'kernel':58s} {'launches/step':>13s} {'ms/step':>9s} {'share':>6s}")
    for k, v in tot.most_common():
        print(f"{k:58s} {cnt[k] / steps:13.1f} {v / steps / 1e3:9.3f} {100 * v / T:5.1f}%")
    print(f"total ms/step (serialised, cold): {T / steps / 1e3:.3f}")


if __name__ == "__main__":
    main()
