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

METRICS = ("gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,"
           "dram__throughput.avg.pct_of_peak_sustained_elapsed")
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
    try:
        return subprocess.run(["git", "rev-parse", "--short=12", "HEAD"], cwd=ROOT, capture_output=True,
                              text=True, timeout=10).stdout.strip() or "unknown"
    except Exception:
        return "unknown"


def gemm_dims(net, shapes, lid: int, batch: int) -> dict:
    """Implicit-GEMM view of a CONV / FC layer: forward M x N x K, wgrad and dgrad."""
    lay = net.layers[lid]
    o, i = shapes[lid], shapes[lay.prev[0]]
    if lay.kind.value == "CONV":
        k = lay.params["k"]
        M, N, K = batch * o[1] * o[2], o[0], k * k * i[0]
        return {"fwd": (M, N, K), "wgrad": (K, N, M), "dgrad": (batch * i[1] * i[2], i[0], k * k * o[0])}
    fan = math.prod(i)
    return {"fwd": (batch, o[0], fan), "wgrad": (fan, o[0], batch), "dgrad": (batch, fan, o[0])}


def is_tensor(name: str) -> bool:
    return any(t in name for t in ("tc_conv", "tc_gemm", "stem_rows_kernel", "stem_wgrad_rows"))


def is_wgrad(name: str) -> bool:
    """Mangled census names: the halo / stem weight-gradient kernels say so;
    tc_conv_tma_kernel<BN, STAGES, MODE, CG> is a weight gradient at MODE 1 or 3;
    tc_gemm_kernel<BN, STAGES, A_MN, B_MN, ...> with both operands MN-major."""
    if "wgrad" in name:
        return True
    if "tc_conv_tma_kernel" in name:
        ints = re.findall(r"Li(\d+)E", name.split("tc_conv_tma_kernel", 1)[1])
        return len(ints) >= 3 and ints[2] in ("1", "3")
    if "tc_gemm_kernel" in name:
        tail = name.split("tc_gemm_kernel", 1)[1]
        flags = re.findall(r"Lb([01])E", tail)
        return len(flags) >= 2 and flags[0] == "1" and flags[1] == "1"
    return False


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
    census = ex.census()
    runs = [ex.profile() for _ in range(5)]
    if args.ncu_region:
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        ex.profile()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    shapes = sn.propagate_shapes(net)
    actions = []
    for i, (names, (ms0, lid, typ)) in enumerate(zip(census, runs[0])):
        a = {"i": i, "layer": lid, "type": TYPES[typ], "kernels": names,
             "ms": statistics.median(r[i][0] for r in runs)}
        if lid >= 0:
            lay = net.layers[lid]
            a["name"], a["kind"] = lay.name, lay.kind.value
            if lay.kind.value in ("CONV", "FC"):
                a["gemm"] = gemm_dims(net, shapes, lid, B)
                a["has_dgrad"] = net.layers[lay.prev[0]].kind.value != "DATA"
        actions.append(a)
    out = {"net": args.net, "batch": B, "pool_bytes": pool, "features": args.features, "precision": args.precision,
           "git_sha": git_sha(), "exec_digest": exec_digest(), "device": torch.cuda.get_device_name(0),
           "kernels_per_step": sum(len(a["kernels"]) for a in actions), "actions": actions,
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


def merge(args) -> None:
    lt = json.load(open(args.json))
    launches = read_ncu(args.csv)
    flat = [(a, k) for a in lt["actions"] for k in a["kernels"]]
    if len(flat) != len(launches):
        sys.exit(f"census has {len(flat)} kernels, ncu region {len(launches)}: not the same iteration")
    def short(ncu_name: str) -> str:
        n = ncu_name.replace("void ", "").replace("unnamed>::", "").replace("(anonymous namespace)::", "")
        m = re.match(r"(?:\w+::)*(\w+)\s*[<(]", n)
        return m.group(1) if m else n
    bad = [(i, short(L["name"]), k) for i, ((a, k), L) in enumerate(zip(flat, launches)) if short(L["name"]) not in k]
    if bad:
        sys.exit(f"census / ncu launch names differ at {len(bad)} launches, first {bad[0]}")
    rows = []
    cls = collections.defaultdict(lambda: {"launches": 0, "s": 0.0, "dram": 0.0, "flops": 0.0})
    for (a, kname), L in zip(flat, launches):
        m = L["m"]
        t = m.get("gpu__time_duration.sum", 0.0)
        dram = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        flops, dims = 0.0, ""
        tensor = is_tensor(kname)
        if tensor and "gemm" in a:
            same = [k for k in a["kernels"] if is_tensor(k)]
            if a["type"] == "bwd":
                wg = [k for k in same if is_wgrad(k)]
                dg = [k for k in same if not is_wgrad(k)]
                part = "wgrad" if is_wgrad(kname) else "dgrad"
                group = wg if part == "wgrad" else dg
            else:
                part, group = "fwd", same
            M, N, K = a["gemm"][part]
            flops = 2.0 * M * N * K / max(1, len(group))
            dims = f"{part} {M}x{N}x{K}" + (f" /{len(group)}" if len(group) > 1 else "")
        key = "tensor (CONV/FC GEMM)" if tensor else "hbm (layer / reduction kernels)"
        c = cls[key]
        c["launches"] += 1
        c["s"] += t
        c["dram"] += dram
        c["flops"] += flops
        rows.append({"i": a["i"], "layer": a.get("name", "-"), "type": a["type"], "kernel": L["name"][:70],
                     "dims": dims, "us": t * 1e6, "flops": flops, "dram": dram,
                     "tflops": flops / t / 1e12 if t and flops else None, "gbs": dram / t / 1e9 if t else None,
                     "tensor_pct": m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                     "dram_pct": m.get("dram__throughput.avg.pct_of_peak_sustained_elapsed")})
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
    md += ["", "| # | layer | phase | kernel | GEMM | us | TF/s | tensor % | DRAM MB | GB/s | DRAM % |",
           "|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        md.append(f"| {r['i']} | {r['layer']} | {r['type']} | `{r['kernel']}` | {r['dims']} | {r['us']:.1f} | "
                  f"{'' if r['tflops'] is None else f'{r['tflops']:.0f}'} | "
                  f"{'' if r['tensor_pct'] is None else f'{r['tensor_pct']:.0f}'} | {r['dram'] / 1e6:.1f} | "
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
