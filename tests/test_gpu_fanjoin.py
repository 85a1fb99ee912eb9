"""The reference's own branchy networks on the GPU: its bundled nested_fan10
fixture and its seeded random_fanjoin property-test generator (memsched
netgen.py:112-171), whose branches often start with an in-place ACT right
after a fork -- the executor gives such a layer its own gradient buffer
(outside the pool) and adds its masked gradient into the forked producer's.

Per net: every feature set yields bit-identical loss and gradients (schedule
soundness), and the fp32-faithful mode matches the CPU oracle (loss 1e-5,
every gradient 1e-4 relative; analytically-zero bias gradients absolutely).
"""

from __future__ import annotations

import math

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ALL = "liveness,offload,cache,recompute=cost-aware,convselect"
SEEDS = list(range(40))


def _case(net, batch=4, seed=0):
    import paper_1801_04380_b200 as sn
    from paper_1801_04380_b200.training import init_parameters
    shp = sn.propagate_shapes(net)
    c, h, w = shp[net.data_id]
    ncls = math.prod(shp[net.terminal_id])
    images = torch.randn(batch, c, h, w, generator=torch.Generator().manual_seed(seed))
    labels = torch.randint(0, ncls, (batch,), generator=torch.Generator().manual_seed(seed + 1))
    return init_parameters(net, seed=seed + 2, head_scale=0.5), images, labels


def _run(net, batch, feats, params, images, labels, **kw):
    import paper_1801_04380_b200 as sn
    from paper_1801_04380_b200.training import Executor
    cfg = sn.SimConfig(pool_bytes=64 << 20, features=sn.parse_features(feats), cost=sn.CostConfig(batch=batch))
    ex = Executor(net, cfg, params=params, **kw)
    ex.set_inputs(images, labels)
    loss, _ = ex.step(update=False)
    g = ex.get("grads")
    ex.close()
    return loss, g


def _check(net):
    from oracle.numerics import forward_backward, relative_error
    params, images, labels = _case(net)
    base_loss, base = _run(net, 4, "none", params, images, labels)
    for feats in ("liveness", "liveness,offload,recompute=memory", ALL):
        loss, g = _run(net, 4, feats, params, images, labels)
        assert loss == base_loss, feats
        assert all(torch.equal(g[l][k], base[l][k]) for l in g for k in ("w", "b")), feats
    loss32, g32 = _run(net, 4, ALL, params, images, labels, precision="fp32")
    ref_loss, ref = forward_backward(net, params, images, labels)
    assert abs(loss32 - ref_loss) <= 1e-5 * abs(ref_loss), (loss32, ref_loss)
    for l in ref:
        wn = ref[l]["w"].double().norm().item()
        assert relative_error(g32[l]["w"], ref[l]["w"]) <= 1e-4, net.layers[l].name
        if ref[l]["b"].double().norm().item() < 1e-4 * wn:
            assert (g32[l]["b"] - ref[l]["b"]).double().norm().item() <= 1e-4 * wn, net.layers[l].name
        else:
            assert relative_error(g32[l]["b"], ref[l]["b"]) <= 1e-4, net.layers[l].name


def test_nested_fan10(cuda):
    from paper_1801_04380_b200.cli import resolve_network
    _check(resolve_network("nested_fan10"))


@pytest.mark.parametrize("seed", SEEDS)
def test_random_fanjoin(cuda, seed):
    from paper_1801_04380_b200 import random_fanjoin
    _check(random_fanjoin(seed))
