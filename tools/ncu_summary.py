"""Summarise an ncu --set full report (.ncu-rep) into a markdown table for profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--algo-json profiles/x.json] > profiles/rNN_ncu_summary.md
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time_us", 1e-3),
    ("dram__bytes_read.sum", "dram_rd_MB", 1e-6),
    ("dram__bytes_write.sum", "dram_wr_MB", 1e-6),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%", 1.0),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_active_%", 1.0),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%", 1.0),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_%", 1.0),
    ("launch__grid_size", "grid", 1.0),
    ("launch__registers_per_thread", "regs", 1.0),
    ("sm__cycles_elapsed.avg.per_second", "sm_GHz", 1e-9),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    idx = {m: hdr.index(m) for m, _, _ in METRICS if m in hdr}
    kn = hdr.index("Kernel Name")
    print("| # | kernel | " + " | ".join(n for m, n, _ in METRICS if m in idx) + " |")
    print("|---|---|" + "---|" * len(idx))
    for i, r in enumerate(rows[2:]):
        name = r[kn].split("(")[0].replace("void ", "").replace("mlora::", "")
        vals = []
        for m, n, s in METRICS:
            if m not in idx:
                continue
            try:
                v = float(r[idx[m]].replace(",", "")) * s
                vals.append(f"{v:.3g}" if v < 1000 else f"{v:.0f}")
            except ValueError:
                vals.append(r[idx[m]])
        print(f"| {i} | `{name}` | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
