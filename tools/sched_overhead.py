"""Where the memory schedule's overhead goes: the bench config (all features,
24 GiB pool) against the unconstrained run (features none, everything
resident), one serial eager iteration each (sn_exec_profile, median of 3),
per-action device ms summed by (layer, phase) and diffed.

    python tools/sched_overhead.py [--net resnet50g] [--out gpurun_out/sched_overhead.json]
"""

from __future__ import annotations

import argparse
import collections
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1801_04380_b200 as sn  # noqa: E402
from paper_1801_04380_b200.training import Executor  # noqa: E402

TYPES = {0: "fwd", 1: "replay", 2: "bwd", 3: "other"}


def profile(net, cfg, batch):
    ex = Executor(net, cfg, device=0, seed=2)
    ex.set_inputs(*bench._inputs(net, batch))
    for _ in range(3):
        ex.step()
    graph_ms = statistics.median(ex.step()[1].step_ms for _ in range(5))
    runs = [ex.profile() for _ in range(3)]
    names = {l.id: l.name for l in net.layers}
    agg = collections.defaultdict(float)
    for i in range(len(runs[0])):
        ms = statistics.median(r[i][0] for r in runs)
        _, lay, typ = runs[0][i]
        agg[(names.get(lay, "-"), TYPES.get(typ, "?"))] += ms
    ex.close()
    return graph_ms, agg, None


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="resnet50g")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--out", default="gpurun_out/sched_overhead.json")
    args = ap.parse_args()
    net = bench.build_net(args.net)
    batch = args.batch
    cost = sn.CostConfig(batch=batch)
    cfg = sn.SimConfig(pool_bytes=bench.DEFAULT_POOL.get(args.net, 24 << 30), features=sn.parse_features(bench.ALL),
                       cost=cost)
    rep = sn.run_simulation(net, cfg)
    ucfg = sn.SimConfig(pool_bytes=rep.baseline_peak_bytes + (256 << 20), features=sn.Features(), cost=cost)
    g_s, a_s, _ = profile(net, cfg, batch)
    g_u, a_u, _ = profile(net, ucfg, batch)
    keys = set(a_s) | set(a_u)
    diff = sorted(((a_s.get(k, 0.0) - a_u.get(k, 0.0), k) for k in keys), reverse=True)
    out = {"net": args.net, "batch": batch, "graph_ms": {"scheduled": g_s, "unconstrained": g_u},
           "serial_ms": {"scheduled": sum(a_s.values()), "unconstrained": sum(a_u.values())},
           "by_phase": {p: {"scheduled": sum(v for (l, q), v in a_s.items() if q == p),
                            "unconstrained": sum(v for (l, q), v in a_u.items() if q == p)}
                        for p in TYPES.values()},
           "diff_ms": [{"layer": k[0], "phase": k[1], "scheduled": round(a_s.get(k, 0.0), 4),
                        "unconstrained": round(a_u.get(k, 0.0), 4), "diff": round(d, 4)} for d, k in diff]}
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps({k: out[k] for k in ("graph_ms", "serial_ms", "by_phase")}))
    for r in out["diff_ms"][:25]:
        print(r)
    for r in out["diff_ms"][-8:]:
        print(r)


if __name__ == "__main__":
    main()
