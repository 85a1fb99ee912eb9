"""Event times (node-by-node replay, median of 5) of the kernels of one
iteration whose name matches a regex -- for A/B runs of kernel knobs.

    SN_POOL_PB=8 python tools/kernel_grep.py 'pool_fwd|pool_bn_stats' [--net resnet50g]
"""

from __future__ import annotations

import argparse
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("regex")
    ap.add_argument("--net", default="resnet50g")
    ap.add_argument("--batch", type=int, default=None)
    args = ap.parse_args()
    import paper_1801_04380_b200 as sn
    from paper_1801_04380_b200.training import Executor
    from paper_1801_04380_b200.profiling import kernel_table
    from bench import ALL, DEFAULT_BATCH, build_net, _inputs
    B = args.batch or DEFAULT_BATCH[args.net]
    net = build_net(args.net)
    cfg = sn.SimConfig(pool_bytes=24 << 30, features=sn.parse_features(ALL), cost=sn.CostConfig(batch=B))
    ex = Executor(net, cfg)
    ex.set_inputs(*_inputs(net, B))
    for _ in range(3):
        _, t = ex.step()
    acts = kernel_table(ex, reps=5)
    tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("SN_"))
    tot = 0.0
    for a in acts:
        for k in a["kernels"]:
            if re.search(args.regex, k["name"]):
                tot += k["us"]
                print(f"{tag:24s} {a.get('name', '-'):>12} {a['type']:>6} {k['us']:8.1f} us  {k['name'][:70]}")
    print(f"{tag:24s} total {tot:.1f} us; graph step {t.step_ms:.3f} ms")
    ex.close()


if __name__ == "__main__":
    main()
