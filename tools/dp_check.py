"""World-1 NCCL data-parallel executor vs the single-replica executor (GPU)."""
import faulthandler
import os
import sys
import traceback

faulthandler.enable()
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1801_04380_b200 as sn  # noqa: E402
from paper_1801_04380_b200 import dp  # noqa: E402
from paper_1801_04380_b200.training import Executor, init_parameters  # noqa: E402

net = sn.load_network("paper_1801_04380_b200/fixtures/alex32.net")
params = init_parameters(net, seed=2, head_scale=0.1)
images = torch.randn(16, 3, 32, 32, generator=torch.Generator().manual_seed(0))
labels = torch.randint(0, 10, (16,), generator=torch.Generator().manual_seed(1))
cfg = sn.SimConfig(pool_bytes=1 << 30, features=sn.parse_features("liveness,offload,cache,recompute=cost-aware,convselect"),
                   cost=sn.CostConfig(batch=16))
print("nccl", dp.nccl_version(), flush=True)
out = []
for use_dp in (False, True):
    try:
        ctx = dp.DPContext(force_comm=True) if use_dp else None
        print("create", use_dp, flush=True)
        ex = Executor(net, cfg, params=params, lr=0.01, dp=ctx, dp_bucket_bytes=1 << 20, use_graph=len(sys.argv) < 2)
        ex.set_inputs(images, labels)
        print("step", use_dp, flush=True)
        losses = [ex.step(update=True)[0] for _ in range(2)]
        print("losses", losses, flush=True)
        out.append((losses, ex.get("params"), ex.get("grads")))
        ex.close()
        if ctx:
            ctx.close()
    except Exception:
        traceback.print_exc()
        sys.exit(1)
(l0, p0, g0), (l1, p1, g1) = out
eq = lambda a, b: all(torch.equal(a[l][k], b[l][k]) for l in a for k in ("w", "b"))  # noqa: E731
print("losses equal", l0 == l1, "params equal", eq(p0, p1), "grads equal", eq(g0, g1))
