"""The numeric oracle restates the network text, shapes, constants and
parameter initialisation on its own (oracle/netdef.py, no product import);
these CPU checks pin that restatement against the product's and the
reference's definitions so the two cannot drift apart silently."""

from __future__ import annotations

import ast
import os

import pytest

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_oracle_never_imports_the_product():
    for fn in os.listdir(os.path.join(ROOT, "oracle")):
        if not fn.endswith(".py"):
            continue
        tree = ast.parse(open(os.path.join(ROOT, "oracle", fn)).read())
        for node in ast.walk(tree):
            mods = []
            if isinstance(node, ast.Import):
                mods = [a.name for a in node.names]
            elif isinstance(node, ast.ImportFrom) and node.module:
                mods = [node.module]
            assert not any(m.startswith("paper_1801_04380_b200") for m in mods), (fn, mods)


@pytest.mark.parametrize("blocks", [(3, 4, 6, 3), (3, 8, 36, 3), (1, 1, 1, 1)])
def test_resnet_text_matches_generator(blocks):
    from oracle import netdef
    from paper_1801_04380_b200.netgen import resnet_text
    assert netdef.resnet_text(*blocks) == resnet_text(*blocks)


@pytest.mark.parametrize("name", ["alex32", "alexnet", "fan12", "resnet50g", "densenet", "inception"])
def test_shapes_params_match_product(name):
    import paper_1801_04380_b200 as sn
    from oracle import netdef
    from paper_1801_04380_b200 import netgen
    from paper_1801_04380_b200.cli import resolve_network
    from paper_1801_04380_b200.training import init_parameters, layer_numerics
    if name == "resnet50g":
        net = netgen.gen_resnet(3, 4, 6, 3)
    elif name == "densenet":
        net = netgen.gen_densenet(blocks=(2, 2), widths=(16, 32))
    elif name == "inception":
        net = netgen.gen_inception(n_a=1, n_b=1, n_c=1)
    else:
        net = resolve_network(name)
    onet = netdef.as_onet(net)
    assert netdef.shapes(onet) == sn.propagate_shapes(net)
    if any(l.kind.value == "SOFTMAX" for l in net.layers) and name != "fan12":
        a, b = init_parameters(net, seed=5, head_scale=0.3), netdef.init_parameters(onet, seed=5, head_scale=0.3)
        assert a.keys() == b.keys()
        assert all(torch.equal(a[l][k], b[l][k]) for l in a for k in ("w", "b"))
    for lay, num in zip(onet.layers, layer_numerics(net)):
        c = netdef.constants(lay)
        assert (c.pool_avg, c.lrn_size, c.lrn_beta, c.lrn_k) == (num.pool_mode == 1, num.lrn_size, pytest.approx(num.lrn_beta), pytest.approx(num.lrn_k))
        assert c.bn_eps == pytest.approx(num.bn_eps) and c.dropout_rate == pytest.approx(num.dropout_rate)


def test_oracle_topological_order_is_valid():
    from oracle import netdef
    from paper_1801_04380_b200.netgen import random_fanjoin
    for seed in range(20):
        onet = netdef.as_onet(random_fanjoin(seed))
        pos = {lid: i for i, lid in enumerate(netdef.topo_order(onet))}
        assert all(pos[p] < pos[l.id] for l in onet.layers for p in l.prev)


def test_bench_reference_arm_loads_no_product_code():
    """bench.py --impl reference runs the oracle and the installed reference
    only: no paper_1801_04380_b200 module (and so no libsnplan / libsnexec)."""
    import subprocess
    import sys
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--net', 'alex32', '--steps', '1', "
            "'--warmup', '1']; runpy.run_path('bench.py', run_name='__main__'); "
            "bad = [m for m in sys.modules if m.startswith('paper_1801_04380_b200')]; "
            "assert not bad, bad")
    proc = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, proc.stderr[-2000:]
    assert '"impl": "reference"' in proc.stdout
