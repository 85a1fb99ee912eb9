"""Run a few eager (non-graph) iterations for ncu / nsys-style launch lists.

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python tools/profile_step.py --steps 2
"""

from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="resnet50g")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--pool-gib", type=float, default=24.0)
    ap.add_argument("--features", default="liveness,offload,cache,recompute=cost-aware,convselect")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--graph", action="store_true")
    ap.add_argument("--order", action="store_true", help="print every action in tape order")
    args = ap.parse_args()
    import torch
    import paper_1801_04380_b200 as sn
    from paper_1801_04380_b200.training import Executor
    from bench import build_net, _inputs
    net = build_net(args.net)
    cfg = sn.SimConfig(pool_bytes=int(args.pool_gib * (1 << 30)), features=sn.parse_features(args.features),
                       cost=sn.CostConfig(batch=args.batch))
    ex = Executor(net, cfg, use_graph=args.graph)
    ex.set_inputs(*_inputs(net, args.batch))
    for _ in range(args.steps):
        loss, t = ex.step()
        print(f"loss {loss:.4f} step {t.step_ms:.2f} ms kernels {t.kernels}", flush=True)
    prof = ex.profile()
    if args.order:
        tot = 0.0
        for i, (ms, lid, typ) in enumerate(prof):
            tot += ms
            name = net.layers[lid].name if lid >= 0 else "-"
            print(f"{i:4d} {name:>14} {['fwd', 'replay', 'bwd', 'copy'][typ]:>6} {ms:8.3f} {tot:8.3f}")
    agg: dict = {}
    for ms, lid, typ in prof:
        if lid >= 0:
            key = (net.layers[lid].name, ["fwd", "replay", "bwd"][typ])
            agg[key] = agg.get(key, 0.0) + ms
    for (name, ph), ms in sorted(agg.items(), key=lambda kv: -kv[1])[:40]:
        print(f"{name:>14} {ph:>6} {ms:8.3f} ms")
    ex.close()


if __name__ == "__main__":
    main()
