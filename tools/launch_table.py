"""Per-launch table of one training iteration, reproducible from one command.

  collect (GPU):  python tools/launch_table.py collect --net resnet50g --out gpurun_out/lt.json [--ncu-region]
      builds the bench config's executor, warms it up, takes the kernel census
      (sn_exec_census: kernel names per tape action) and the serial per-action
      event times (sn_exec_profile, median of 5).  With --ncu-region one more
      serial iteration runs between cudaProfilerStart/Stop, for
        ncu --profile-from-start off --metrics <METRICS> --csv --log-file X.csv \\
            python tools/launch_table.py collect ... --ncu-region
  merge (CPU):    python tools/launch_table.py merge gpurun_out/lt.json gpurun_out/X.csv --tag r02_resnet50g
      aligns the ncu launch list with the census (same order, names checked),
      and writes profiles/<tag>_launches.md (layer, kernel, GEMM M x N x K,
      FLOPs or DRAM bytes, us, TF/s or GB/s, tensor %, DRAM %) and
      profiles/<tag>_step_traffic.json, stamped with the source digest of the
      libsnexec.so that produced it (bench.py refuses a traffic file whose
      digest differs from the library it runs).
"""

from __future__ import annotations

import argparse
import collections
import csv
import json
import math
import os
import re
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1801_04380_b200.profiling import is_tensor, is_wgrad  # noqa: E402

METRICS = ("gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,"
           "dram__throughput.avg.pct_of_peak_sustained_elapsed,"
           "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed")
# the last metric: tensor-core operand reads from shared memory (% of the SMEM
# bandwidth the tensor pipe can draw) -- what bounds the N = 64 convolutions
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6,
         "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "%": 1.0, "": 1.0}
TYPES = ["fwd", "replay", "bwd", "other"]


def exec_digest() -> str:
    p = os.path.join(ROOT, "paper_1801_04380_b200", "_lib", "libsnexec.so.sha")
    try:
        return open(p).read().strip()
    except OSError:
        return "unknown"


def git_sha() -> str:
    """HEAD of the tree this runs from; on the GPU box (a snapshot without .git)
    the .graft_head file written next to the sources before the call."""
    try:
        out = subprocess.run(["git", "rev-parse", "--short=12", "HEAD"], cwd=ROOT, capture_output=True,
                             text=True, timeout=10).stdout.strip()
        if out:
            return out
    except Exception:
        pass
    try:
        return open(os.path.join(ROOT, ".graft_head")).read().strip()[:12] + " (+ working tree)"
    except OSError:
        return "unknown"


def collect(args) -> None:
    import torch
    import paper_1801_04380_b200 as sn
    from bench import DEFAULT_BATCH, DEFAULT_POOL, GiB, build_net, _inputs
    from paper_1801_04380_b200.training import Executor
    net = build_net(args.net)
    B = args.batch or DEFAULT_BATCH[args.net]
    pool = int(args.pool_gib * GiB) if args.pool_gib else DEFAULT_POOL.get(args.net, 24 * GiB)
    cfg = sn.SimConfig(pool_bytes=pool, features=sn.parse_features(args.features), cost=sn.CostConfig(batch=B))
    ex = Executor(net, cfg, precision=args.precision)
    ex.set_inputs(*_inputs(net, B))
    for _ in range(3):
        ex.step(update=False)
    from paper_1801_04380_b200.profiling import kernel_table
    actions = kernel_table(ex, reps=5)  # census + per-kernel event times + FLOP attribution
    runs = [ex.profile() for _ in range(5)]
    if args.ncu_region:
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        ex.profile()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    for a, r in zip(actions, zip(*runs)):
        a["ms"] = statistics.median(x[0] for x in r)
        a["kernel_names"] = [k["name"] for k in a["kernels"]]
    out = {"net": args.net, "batch": B, "pool_bytes": pool, "features": args.features, "precision": args.precision,
           "git_sha": git_sha(), "exec_digest": exec_digest(), "device": torch.cuda.get_device_name(0),
           "kernels_per_step": sum(len(a["kernels"]) for a in actions), "actions": actions,
           "kernel_event_us_per_step": sum(k["us"] for a in actions for k in a["kernels"]),
           "serial_step_ms": statistics.median(sum(x[0] for x in r) for r in runs)}
    ex.close()
    with open(args.out, "w") as fh:
        json.dump(out, fh)
    print(f"{args.out}: {len(actions)} actions, {out['kernels_per_step']} kernels, "
          f"serial step {out['serial_step_ms']:.3f} ms", flush=True)


def read_ncu(path: str) -> list[dict]:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hi]
    ix = {h: i for i, h in enumerate(hdr)}
    launches: dict[int, dict] = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) != len(hdr):
            continue
        d = launches.setdefault(int(r[ix["ID"]]), {"name": r[ix["Kernel Name"]], "m": {}})
        val = r[ix["Metric Value"]].replace(",", "")
        try:
            d["m"][r[ix["Metric Name"]]] = float(val) * UNITS.get(r[ix["Metric Unit"]], 1.0)
        except ValueError:
            pass
    return list(launches.values())


BULK = 50e6  # bytes per launch


def merge(args) -> None:
    lt = json.load(open(args.json))
    launches = read_ncu(args.csv)
    flat = [(a, k["name"]) for a in lt["actions"] for k in a["kernels"]]
    kinfo = [k for a in lt["actions"] for k in a["kernels"]]
    if len(flat) != len(launches):
        sys.exit(f"census has {len(flat)} kernels, ncu region {len(launches)}: not the same iteration")
    ev_cls = collections.defaultdict(float)
    for a in lt["actions"]:
        for k in a["kernels"]:
            ev_cls["tensor" if is_tensor(k["name"]) else "hbm"] += k["us"]
    def short(ncu_name: str) -> str:
        n = ncu_name.replace("void ", "").replace("unnamed>::", "").replace("(anonymous namespace)::", "")
        m = re.match(r"(?:\w+::)*(\w+)\s*[<(]", n)
        return m.group(1) if m else n
    bad = [(i, short(L["name"]), k) for i, ((a, k), L) in enumerate(zip(flat, launches)) if short(L["name"]) not in k]
    if bad:
        sys.exit(f"census / ncu launch names differ at {len(bad)} launches, first {bad[0]}")
    rows = []
    cls = collections.defaultdict(lambda: {"launches": 0, "s": 0.0, "dram": 0.0, "flops": 0.0})
    # the bulk HBM launches (>= BULK bytes each): where the layer kernels' roofline is decided;
    # the many short launches (finalisers, tile statistics, weight transposes) are latency
    bulk = {"launches": 0, "s": 0.0, "dram": 0.0, "flops": 0.0, "flat": []}
    for fi, (((a, kname), L), ki) in enumerate(zip(zip(flat, launches), kinfo)):
        m = L["m"]
        t = m.get("gpu__time_duration.sum", 0.0)
        dram = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        flops, tensor = ki["flops"], is_tensor(kname)
        dims = ""
        if flops:
            M, N, K = a["gemm"][ki["part"]]
            nk = sum(1 for k in a["kernels"] if k.get("part") == ki["part"])
            dims = f"{ki['part']} {M}x{N}x{K}" + (f" /{nk}" if nk > 1 else "")
        key = "tensor (CONV/FC GEMM)" if tensor else "hbm (layer / reduction kernels)"
        c = cls[key]
        c["launches"] += 1
        c["s"] += t
        c["dram"] += dram
        c["flops"] += flops
        if not tensor and dram >= BULK:
            bulk["launches"] += 1
            bulk["s"] += t
            bulk["dram"] += dram
            bulk["flat"].append(fi)
        rows.append({"i": a["i"], "layer": a.get("name", "-"), "type": a["type"], "kernel": L["name"][:70],
                     "dims": dims, "us": t * 1e6, "ev_us": ki["us"], "flops": flops, "dram": dram,
                     "tflops": flops / t / 1e12 if t and flops else None, "gbs": dram / t / 1e9 if t else None,
                     "tensor_pct": m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                     "dram_pct": m.get("dram__throughput.avg.pct_of_peak_sustained_elapsed"),
                     "tcsmem_pct": m.get("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed")})
    tag = args.tag
    md = [f"# Per-launch table: {lt['net']} b{lt['batch']} ({lt['features']}, {lt['precision']})", "",
          f"Source: `tools/launch_table.py collect` + ncu `--profile-from-start off --metrics {METRICS}` over one "
          f"serial eager iteration (weight gradients on the compute stream; cold, serialised launches: compare "
          f"shares, not absolutes).  git {lt['git_sha']}, libsnexec digest `{lt['exec_digest'][:16]}`, "
          f"{lt['device']}.  {len(rows)} launches; serial event time {lt['serial_step_ms']:.3f} ms.", "",
          "| class | launches | ncu time ms | share | DRAM GB | GB/s | TFLOP | TF/s |", "|---|---|---|---|---|---|---|---|"]
    tot = sum(c["s"] for c in cls.values())
    for k, c in sorted(cls.items()):
        md.append(f"| {k} | {c['launches']} | {c['s'] * 1e3:.3f} | {c['s'] / tot:.3f} | {c['dram'] / 1e9:.3f} | "
                  f"{c['dram'] / c['s'] / 1e9:.0f} | {c['flops'] / 1e12:.4f} | "
                  f"{(c['flops'] / c['s'] / 1e12) if c['flops'] else 0:.1f} |")
    if bulk["launches"]:
        md.append(f"| of which hbm launches moving >= {BULK / 1e6:.0f} MB | {bulk['launches']} | {bulk['s'] * 1e3:.3f} | "
                  f"{bulk['s'] / tot:.3f} | {bulk['dram'] / 1e9:.3f} | {bulk['dram'] / bulk['s'] / 1e9:.0f} | | |")
    md += ["", "`us` = ncu gpu__time_duration (cold); `ev us` = CUDA-event time of the same kernel in a node-by-node "
           "replay of the iteration (warm, `sn_exec_kernel_times`, median of 5); TF/s from the ncu time.", "",
           "`TC smem %` = tensor-core operand reads from shared memory, % of their peak "
           "(l1tex__data_pipe_tc_wavefronts_mem_shared): near 80-90 % a convolution is bound by its SMEM operand "
           "traffic, not by the MMA rate.", "",
           "| # | layer | phase | kernel | GEMM | us | ev us | TF/s | tensor % | TC smem % | DRAM MB | GB/s | DRAM % |",
           "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        md.append(f"| {r['i']} | {r['layer']} | {r['type']} | `{r['kernel']}` | {r['dims']} | {r['us']:.1f} | "
                  f"{r['ev_us']:.1f} | "
                  f"{'' if r['tflops'] is None else f'{r['tflops']:.0f}'} | "
                  f"{'' if r['tensor_pct'] is None else f'{r['tensor_pct']:.0f}'} | "
                  f"{'' if not r['tcsmem_pct'] else f'{r['tcsmem_pct']:.0f}'} | {r['dram'] / 1e6:.1f} | "
                  f"{'' if r['gbs'] is None else f'{r['gbs']:.0f}'} | "
                  f"{'' if r['dram_pct'] is None else f'{r['dram_pct']:.0f}'} |")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{tag}_launches.md"), "w") as fh:
        fh.write("\n".join(md) + "\n")
    traffic = {"net": lt["net"], "batch": lt["batch"], "features": lt["features"], "precision": lt["precision"],
               "git_sha": lt["git_sha"], "exec_digest": lt["exec_digest"], "launches": len(rows),
               "per_step": {("conv_fc_gemm" if k.startswith("tensor") else "hbm_layers"):
                            {"launches": c["launches"], "dram_bytes_per_step": c["dram"], "ncu_ms": c["s"] * 1e3,
                             "algorithmic_tflop": c["flops"] / 1e12} for k, c in cls.items()}}
    traffic["per_step"]["hbm_bulk"] = {"min_bytes_per_launch": BULK, "launches": bulk["launches"],
                                       "dram_bytes_per_step": bulk["dram"], "ncu_ms": bulk["s"] * 1e3,
                                       "flat_kernel_indices": bulk["flat"]}
    with open(os.path.join(ROOT, "profiles", f"{tag}_step_traffic.json"), "w") as fh:
        json.dump(traffic, fh, indent=1)
    print(f"profiles/{tag}_launches.md, profiles/{tag}_step_traffic.json")


def main() -> None:
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    c = sub.add_parser("collect")
    c.add_argument("--net", default="resnet50g")
    c.add_argument("--batch", type=int, default=None)
    c.add_argument("--pool-gib", type=float, default=None)
    c.add_argument("--features", default="liveness,offload,cache,recompute=cost-aware,convselect")
    c.add_argument("--precision", default="tf32")
    c.add_argument("--out", required=True)
    c.add_argument("--ncu-region", action="store_true")
    m = sub.add_parser("merge")
    m.add_argument("json")
    m.add_argument("csv")
    m.add_argument("--tag", required=True)
    args = ap.parse_args()
    collect(args) if args.cmd == "collect" else merge(args)


if __name__ == "__main__":
    main()
