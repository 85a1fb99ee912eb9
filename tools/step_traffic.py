"""Per-kernel-class DRAM traffic and time of the launches in an ncu metrics
CSV (ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
--csv --log-file X python tools/profile_step.py --steps 1), per training step
(profile_step runs two iterations: --iterations 2).

    python tools/step_traffic.py gpurun_out/traffic_step.csv [--iterations 2] [--json out.json]
"""
from __future__ import annotations

import argparse
import collections
import csv
import json

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6,
         "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}


def klass(name: str) -> str:
    if "tc_conv" in name or "tc_gemm" in name:
        return "conv_fc_gemm"
    return "hbm_layers"


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--iterations", type=int, default=2)
    ap.add_argument("--json")
    args = ap.parse_args()
    rows = list(csv.reader(open(args.csv)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hi]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = collections.defaultdict(lambda: {"launches": 0, "dram_bytes": 0.0, "ms": 0.0})
    for r in rows[hi + 1:]:
        if len(r) != len(hdr):
            continue
        k = klass(r[ix["Kernel Name"]])
        m, u = r[ix["Metric Name"]], r[ix["Metric Unit"]]
        v = float(r[ix["Metric Value"]].replace(",", "")) * UNITS[u]
        if m.startswith("dram__bytes"):
            agg[k]["dram_bytes"] += v
        elif m == "gpu__time_duration.sum":
            agg[k]["ms"] += v * 1e3
            agg[k]["launches"] += 1
    out = {k: {"launches_per_step": v["launches"] / args.iterations,
               "dram_bytes_per_step": v["dram_bytes"] / args.iterations,
               "ms_per_step_serialised": v["ms"] / args.iterations} for k, v in agg.items()}
    print(json.dumps(out, indent=1))
    if args.json:
        with open(args.json, "w") as fh:
            json.dump({"source": args.csv, "per_step": out}, fh, indent=1)


if __name__ == "__main__":
    main()
