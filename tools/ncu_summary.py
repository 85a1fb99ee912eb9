"""Summarise ncu reports / launch lists into profiles/ (tracked evidence).

    python tools/ncu_summary.py report gpurun_out/prof.ncu-rep  > profiles/x.md
    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/y.md
"""

from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor %"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "TC smem %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("dram__bytes_read.sum", "DRAM rd"),
    ("dram__bytes_write.sum", "DRAM wr"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "regs"),
    ("launch__shared_mem_per_block_dynamic", "smem"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
]


def report(path: str) -> None:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    print(f"# ncu --set full summary: `{path}`\n")
    print("| kernel | " + " | ".join(k[1] for k in KEYS) + " |")
    print("|---|" + "---|" * len(KEYS))
    for r in rows[2:]:
        name = r[idx["Kernel Name"]]
        short = name.split("(")[0].replace("void ", "")[:60]
        cells = []
        for k, _ in KEYS:
            v = r[idx[k]] if k in idx else "-"
            u = units[idx[k]] if k in idx else ""
            cells.append(f"{v} {u}".strip())
        print(f"| `{short}` | " + " | ".join(cells) + " |")


def launches(path: str) -> None:
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    idx = {h: i for i, h in enumerate(hdr)}
    agg: dict[str, float] = collections.defaultdict(float)
    cnt: collections.Counter = collections.Counter()
    for r in rows[start + 1:]:
        if len(r) < len(hdr) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[idx["Kernel Name"]].split("(")[0].replace("void ", "")[:70]
        unit = r[idx["Metric Unit"]]
        v = float(r[idx["Metric Value"]].replace(",", ""))
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(unit, 1e-6)
        agg[name] += v * scale
        cnt[name] += 1
    total = sum(agg.values())
    print(f"# launch list (ncu gpu__time_duration, cold-cache, serialised): `{path}`\n")
    print(f"total {total:.3f} ms over {sum(cnt.values())} launches\n")
    print("| ms | share | launches | kernel |")
    print("|---:|---:|---:|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
        print(f"| {v:.3f} | {100 * v / total:.1f}% | {cnt[k]} | `{k}` |")


if __name__ == "__main__":
    {"report": report, "launches": launches}[sys.argv[1]](sys.argv[2])
