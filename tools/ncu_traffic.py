"""profiles/ncu_traffic.json from an ncu --set full capture of one bench step:
the DRAM bytes (read + write) per launch of the dominant kernel (the forward base
GEMM, mlora_base_pair_kernel<6, false>) and its algorithmic bytes, so bench.py's
roofline.traffic is the measured figure of the shipped build.

    python tools/ncu_traffic.py gpurun_out/step_full.ncu-rep [rows=8192]
"""
import csv
import io
import json
import subprocess
import sys
import time

LLAMA7B = [("q", 4096, 4096), ("k", 4096, 4096), ("v", 4096, 4096), ("o", 4096, 4096), ("gate", 11008, 4096),
           ("up", 11008, 4096), ("down", 4096, 11008)]


def main(path, rows=8192, R=64):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--print-units", "base"], capture_output=True,
                         text=True, check=True).stdout
    rs = list(csv.reader(io.StringIO(out)))
    hdr, body = rs[0], [r for r in rs[2:] if r]
    kn, rd, wr, tm = (hdr.index(c) for c in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                               "gpu__time_duration.sum"))
    fwd = [r for r in body if "mlora_base_pair_kernel" in r[kn] and ("<6, false" in r[kn] or "<6, 0" in r[kn])]
    if len(fwd) < len(LLAMA7B):
        raise SystemExit(f"expected {len(LLAMA7B)} forward base GEMM launches, found {len(fwd)}")
    fwd = fwd[:len(LLAMA7B)]  # the capture starts at a step boundary: q, k, v, gate, up, o, down
    per = []
    for (name, d, k), r in zip(LLAMA7B, fwd):
        algo = 2 * (rows * k + d * k + d * R + rows * R + rows * d)  # X, W0, B_cat, H read once; Y written once
        per.append({"projection": name, "dram_bytes": float(r[rd]) + float(r[wr]), "algorithmic_bytes": algo,
                    "time_us": float(r[tm]) / 1e3})
    mean = sum(p["dram_bytes"] for p in per) / len(per)
    algo = sum(p["algorithmic_bytes"] for p in per) / len(per)
    doc = {"base_fwd_dram_bytes_per_launch": round(mean), "base_fwd_algorithmic_bytes_per_launch": round(algo),
           "ratio": round(mean / algo, 3), "per_launch": per, "source": path,
           "how": "ncu --set full --clock-control none -k regex:mlora on python bench.py --steps 1 --warmup 3; "
                  "dram__bytes_read.sum + dram__bytes_write.sum of the 7 forward base GEMM launches of one step",
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    with open("profiles/ncu_traffic.json", "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps({k: doc[k] for k in ("base_fwd_dram_bytes_per_launch", "base_fwd_algorithmic_bytes_per_launch",
                                          "ratio")}))


if __name__ == "__main__":
    main(sys.argv[1], *[int(a) for a in sys.argv[2:]])
