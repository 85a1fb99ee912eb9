"""Where a config's step goes: every kernel of one iteration event-timed in a
node-by-node replay (profiling.kernel_table), aggregated by layer kind / phase
and by kernel name, plus the tensor kernels' TF/s.

    python tools/kernel_top.py --net densenet121s [--batch 256]
"""

from __future__ import annotations

import argparse
import collections
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="resnet50g")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--pool-gib", type=float, default=24.0)
    ap.add_argument("--top", type=int, default=30)
    args = ap.parse_args()
    import paper_1801_04380_b200 as sn
    from paper_1801_04380_b200.training import Executor
    from paper_1801_04380_b200.profiling import kernel_table
    from bench import ALL, DEFAULT_BATCH, build_net, _inputs
    B = args.batch or DEFAULT_BATCH[args.net]
    net = build_net(args.net)
    cfg = sn.SimConfig(pool_bytes=int(args.pool_gib * (1 << 30)), features=sn.parse_features(ALL),
                       cost=sn.CostConfig(batch=B))
    ex = Executor(net, cfg)
    ex.set_inputs(*_inputs(net, B))
    for _ in range(3):
        _, t = ex.step()
    print(f"{args.net} b{B}: graph step {t.step_ms:.3f} ms, {t.kernels} kernels")
    acts = kernel_table(ex, reps=3)
    by_kind = collections.Counter()
    by_name = collections.Counter()
    cnt = collections.Counter()
    fl = collections.Counter()
    tot = 0.0
    for a in acts:
        kind = a.get("kind", "-")
        for k in a["kernels"]:
            nm = re.sub(r"_GLOBAL__N__[0-9a-f_]+|\(.*", "", k["name"])
            nm = re.sub(r"^_ZN2sn\d+\w*?(?=[a-z_]+_kernel|tc_|colred|bn_|pool|splitk|stem|transpose|softmax)", "", nm)[:60]
            by_kind[(kind, a["type"])] += k["us"]
            by_name[nm] += k["us"]
            cnt[nm] += 1
            fl[nm] += k.get("flops", 0.0)
            tot += k["us"]
    print(f"serial kernel time {tot / 1e3:.3f} ms")
    print("\nby layer kind / phase (ms):")
    for (kind, ph), us in by_kind.most_common():
        print(f"  {kind:>8} {ph:>6} {us / 1e3:8.3f}  {100 * us / tot:5.1f} %")
    print(f"\ntop {args.top} kernels by total event time:")
    for nm, us in by_name.most_common(args.top):
        tf = f"{fl[nm] / (us / 1e6) / 1e12:7.1f} TF/s" if fl[nm] else ""
        print(f"  {us / 1e3:8.3f} ms {cnt[nm]:5d}x {100 * us / tot:5.1f} % {tf:>13}  {nm}")
    ex.close()


if __name__ == "__main__":
    main()
