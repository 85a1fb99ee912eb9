"""Diagnostic: run the executor on small configs and print per-layer parity.

    python tools/gpu_check.py [alex32|resnet|alexnet]
"""

from __future__ import annotations

import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1801_04380_b200 as sn  # noqa: E402
from paper_1801_04380_b200.training import Executor, init_parameters  # noqa: E402
from oracle.numerics import forward_backward, relative_error  # noqa: E402

ALL = "liveness,offload,cache,recompute=cost-aware,convselect"


def run(net, batch, pool, feats, params, images, labels, graph=True, elide=True, quiet=False):
    cfg = sn.SimConfig(pool_bytes=pool, features=sn.parse_features(feats), cost=sn.CostConfig(batch=batch))
    ex = Executor(net, cfg, params=params, use_graph=graph, elide_backups=elide)
    ex.set_inputs(images, labels)
    t0 = time.time()
    loss, t = ex.step(update=False)
    wall = time.time() - t0
    g = ex.get("grads")
    if not quiet:
        print(f"  [{feats:<55}] graph={int(graph)} elide={int(elide)} loss={loss:.6f} "
              f"step={t.step_ms:.3f}ms wall={wall:.2f}s kernels={t.kernels} d2h={t.d2h_bytes} h2d={t.h2d_bytes} "
              f"peak={ex.report.peak_bytes} hw={ex.report.pool_high_water_bytes} "
              f"evict={ex.report.evictions} demand={ex.report.demand_transfer_count}", flush=True)
    ex.close()
    return loss, g


def compare(net, g, ref):
    worst = 0.0
    for lid, r in ref.items():
        for k in ("w", "b"):
            e = relative_error(g[lid][k], r[k])
            worst = max(worst, e)
            if e > 1e-2:
                print(f"    layer {net.layers[lid].name:>12} {k}: rel err {e:.3e}")
    return worst


def bitwise(a, b):
    return all(torch.equal(a[l][k], b[l][k]) for l in a for k in ("w", "b"))


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "alex32"
    torch.manual_seed(0)
    if which == "alex32":
        net = sn.load_network(os.path.join(ROOT, "paper_1801_04380_b200", "fixtures", "alex32.net"))
        batch, pool, hw, C = 16, 1 << 30, 32, 10
    elif which == "alexnet":
        net = sn.load_network(os.path.join(ROOT, "paper_1801_04380_b200", "fixtures", "alexnet.net"))
        batch, pool, hw, C = 32, 4 << 30, 227, 1000
    else:
        from paper_1801_04380_b200.netgen import gen_resnet
        net = gen_resnet(3, 4, 6, 3)
        batch, pool, hw, C = 8, 24 << 30, 224, 1000
    params = init_parameters(net, seed=2)
    images = torch.randn(batch, 3, hw, hw, generator=torch.Generator().manual_seed(0))
    labels = torch.randint(0, C, (batch,), generator=torch.Generator().manual_seed(1))
    t0 = time.time()
    acts: dict = {}
    ref_loss, ref = forward_backward(net, params, images, labels, activations=acts)
    print(f"{which}: oracle loss {ref_loss:.6f} ({time.time() - t0:.1f}s)", flush=True)
    acts64: dict = {}
    loss64, ref64 = forward_backward(net, params, images, labels, activations=acts64, dtype=torch.float64)
    acts_t: dict = {}
    loss_t, ref_t = forward_backward(net, params, images, labels, activations=acts_t, tf32=True)
    print(f"  oracle fp64 loss {loss64:.6f}, tf32-emulated loss {loss_t:.6f}", flush=True)
    cfg = sn.SimConfig(pool_bytes=pool, features=sn.parse_features("none"), cost=sn.CostConfig(batch=batch))
    ex = Executor(net, cfg, params=params, use_graph=False)
    ex.set_inputs(images, labels)
    ex.step(update=False)
    print("  per-layer activation rel err: gpu-vs-fp32 | gpu-vs-fp64 | fp32-vs-fp64 | gpu-vs-tf32emu", flush=True)
    for lid in sn.forward_order(net):
        if net.layers[lid].kind is sn.LayerKind.DATA:
            continue
        a = ex.read_activation(lid)
        r, r64, rt = acts[lid].reshape(a.shape), acts64[lid].reshape(a.shape), acts_t[lid].reshape(a.shape)
        print(f"    {net.layers[lid].name:>14} {relative_error(a, r):.2e} | {relative_error(a, r64):.2e} | "
              f"{relative_error(r, r64):.2e} | {relative_error(a, rt):.2e}", flush=True)
    g = ex.get("grads")
    ex.close()
    print("  grad rel err: gpu-vs-fp64 | fp32-vs-fp64 | gpu-vs-tf32emu")
    for lid in ref:
        print(f"    {net.layers[lid].name:>14} w {relative_error(g[lid]['w'], ref64[lid]['w']):.2e} | "
              f"{relative_error(ref[lid]['w'], ref64[lid]['w']):.2e} | {relative_error(g[lid]['w'], ref_t[lid]['w']):.2e}")
    base_loss, base = run(net, batch, pool, "none", params, images, labels, graph=False)
    print(f"  worst rel err vs oracle (none, eager): {compare(net, base, ref):.3e}", flush=True)
    for feats in ["none", "liveness", "liveness,offload", "liveness,offload,recompute=speed",
                  "liveness,offload,recompute=memory", "cache,recompute=cost-aware", ALL]:
        loss, g = run(net, batch, pool, feats, params, images, labels)
        print(f"    bitwise == none/eager: {bitwise(g, base)}  loss equal: {loss == base_loss}", flush=True)
    loss, g = run(net, batch, pool, ALL, params, images, labels, elide=False)
    print(f"    parity-mode copies bitwise: {bitwise(g, base)}", flush=True)


if __name__ == "__main__":
    main()
