"""End-to-end parity of the B200 executor (through libsnexec.so).

1. Numerics vs the CPU fp32 oracle (oracle/numerics.py): loss and every
   parameter gradient.  The GPU contracts CONV/FC in tf32 (10-bit mantissa,
   fp32 accumulate).  Stated tolerances (classifier scaled by 0.1 so the
   softmax is not saturated, see training.init_parameters):
     * smooth net (no ReLU / max-pool / dropout masks): loss rel. err <= 1e-3,
       every parameter gradient rel. Frobenius err <= 5e-3;
     * nets with masks (alex32, ResNet-50g): loss rel. err <= 2e-3 (5e-3 for
       ResNet); gradients within 3x (+5e-3) of how far tf32 rounding alone moves
       the fp32 gradients (ReLU masks and max-pool argmaxes flip on near-ties),
       measured per case with the oracle's tf32 emulation.
2. Schedule soundness: every feature set (liveness, offload, cache, the three
   recompute policies, convselect, tight pools with evictions and demand
   fetches, parity-mode copy-outs, eager vs CUDA graph) yields BIT-IDENTICAL
   loss and gradients to the unscheduled run.  Any read of a freed, evicted,
   overwritten or not-yet-fetched tensor would break this.
"""

from __future__ import annotations

import os

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ALL = "liveness,offload,cache,recompute=cost-aware,convselect"
FEATURES = ["none", "liveness", "liveness,offload", "liveness,offload,recompute=speed",
            "liveness,offload,recompute=memory", "cache,recompute=cost-aware", ALL]


def _sn():
    import paper_1801_04380_b200 as sn
    return sn


def _fixture(name):
    sn = _sn()
    return sn.load_network(os.path.join(ROOT, "paper_1801_04380_b200", "fixtures", f"{name}.net"))


def _inputs(net, batch, seed=0):
    sn = _sn()
    import math
    c, h, w = sn.propagate_shapes(net)[net.data_id]
    ncls = math.prod(sn.propagate_shapes(net)[net.terminal_id])
    images = torch.randn(batch, c, h, w, generator=torch.Generator().manual_seed(seed))
    labels = torch.randint(0, ncls, (batch,), generator=torch.Generator().manual_seed(seed + 1))
    return images, labels


def _run(net, batch, pool, feats, params, images, labels, **kw):
    sn = _sn()
    from paper_1801_04380_b200.training import Executor
    cfg = sn.SimConfig(pool_bytes=pool, features=sn.parse_features(feats), cost=sn.CostConfig(batch=batch))
    ex = Executor(net, cfg, params=params, **kw)
    ex.set_inputs(images, labels)
    loss, timing = ex.step(update=False)
    grads = ex.get("grads")
    rep = ex.report
    ex.close()
    return loss, grads, rep, timing


def _bitwise(a, b):
    return all(torch.equal(a[l][k], b[l][k]) for l in a for k in ("w", "b"))


@pytest.fixture(scope="module")
def alex32_case():
    from paper_1801_04380_b200.training import init_parameters
    net = _fixture("alex32")
    params = init_parameters(net, seed=2, head_scale=0.1)
    images, labels = _inputs(net, 16)
    return net, params, images, labels


SMOOTH32 = """
layer data DATA c=3 h=32 w=32
layer conv1 CONV out=64 k=5 s=1 p=2
layer bn1 BN
layer lrn1 LRN
layer pool1 POOL k=3 s=2 mode=avg
layer conv2 CONV out=192 k=5 s=1 p=2
layer bn2 BN
layer pool2 POOL k=3 s=2 mode=avg
layer conv3 CONV out=384 k=3 s=1 p=1
layer bn3 BN
layer conv4 CONV out=384 k=3 s=1 p=1
layer join4 JOIN
layer fc1 FC out=256
layer drop1 DROPOUT rate=0.0
layer fc2 FC out=10
layer softmax SOFTMAX
edge data conv1
edge conv1 bn1
edge bn1 lrn1
edge lrn1 pool1
edge pool1 conv2
edge conv2 bn2
edge bn2 pool2
edge pool2 conv3
edge conv3 bn3
edge bn3 conv4
edge conv4 join4
edge bn3 join4
edge join4 fc1
edge fc1 drop1
edge drop1 fc2
edge fc2 softmax
"""


def test_smooth_net_matches_cpu_oracle_tightly(cuda):
    """No ReLU / max-pool / dropout masks: the only discrepancy left is tf32
    rounding, so every CONV/BN/LRN/avg-POOL/JOIN/FC/SOFTMAX backward kernel is
    checked to 5e-3 against the fp32 oracle."""
    sn = _sn()
    from paper_1801_04380_b200.training import init_parameters
    from oracle.numerics import forward_backward, relative_error
    net = sn.parse_network(SMOOTH32, name="smooth32")
    params = init_parameters(net, seed=4, head_scale=0.1)
    images, labels = _inputs(net, 16)
    loss, grads, rep, _ = _run(net, 16, 1 << 30, ALL, params, images, labels)
    ref_loss, ref = forward_backward(net, params, images, labels)
    assert abs(loss - ref_loss) <= 1e-3 * abs(ref_loss), (loss, ref_loss)
    # A CONV bias feeding a training-mode BN has an exactly-zero gradient (BN
    # removes any per-channel shift); both sides hold only rounding noise there,
    # so it is compared absolutely against the layer's weight-gradient scale.
    errs = {}
    for l in ref:
        lay = net.layers[l]
        bn_fed = lay.kind is sn.LayerKind.CONV and net.layers[lay.next[0]].kind is sn.LayerKind.BN
        errs[(lay.name, "w")] = relative_error(grads[l]["w"], ref[l]["w"])
        if bn_fed:
            scale = ref[l]["w"].norm().item()
            errs[(lay.name, "b")] = (grads[l]["b"] - ref[l]["b"]).norm().item() / scale
        else:
            errs[(lay.name, "b")] = relative_error(grads[l]["b"], ref[l]["b"])
    assert max(errs.values()) <= 5e-3, sorted(errs.items(), key=lambda kv: -kv[1])[:4]


def _sensitivity(net, params, images, labels):
    """How far tf32 rounding alone moves the fp32 gradients (CPU emulation):
    ReLU masks and max-pool argmaxes flip on near-ties, so a tf32 run cannot
    be closer to fp32 than this, whatever the kernels do."""
    from oracle.numerics import forward_backward, relative_error
    _, ref = forward_backward(net, params, images, labels)
    _, emu = forward_backward(net, params, images, labels, tf32=True)
    return ref, max(relative_error(emu[l][k], ref[l][k]) for l in ref for k in ("w", "b"))


def test_alex32_matches_cpu_oracle(cuda, alex32_case):
    from oracle.numerics import forward_backward, relative_error
    net, params, images, labels = alex32_case
    loss, grads, rep, _ = _run(net, 16, 1 << 30, ALL, params, images, labels)
    assert rep.peak_bytes == rep.min_pool_bytes == 16777216
    ref_loss, _ = forward_backward(net, params, images, labels)
    assert abs(loss - ref_loss) <= 2e-3 * abs(ref_loss)
    ref, sens = _sensitivity(net, params, images, labels)
    worst = max(relative_error(grads[l][k], ref[l][k]) for l in ref for k in ("w", "b"))
    assert worst <= 3 * sens + 5e-3, (worst, sens)


@pytest.mark.parametrize("feats", FEATURES[1:])
def test_alex32_feature_sets_are_bit_identical(cuda, alex32_case, feats):
    net, params, images, labels = alex32_case
    base_loss, base, _, _ = _run(net, 16, 1 << 30, "none", params, images, labels)
    loss, grads, _, _ = _run(net, 16, 1 << 30, feats, params, images, labels)
    assert loss == base_loss
    assert _bitwise(grads, base)


@pytest.mark.parametrize("pool", [16777216, 17 << 20, 20 << 20])
@pytest.mark.parametrize("feats", [ALL, "cache,recompute=memory", "cache,recompute=speed,convselect"])
def test_alex32_tight_pools_are_bit_identical(cuda, alex32_case, pool, feats):
    net, params, images, labels = alex32_case
    _, base, _, _ = _run(net, 16, 1 << 30, "none", params, images, labels)
    try:
        _, grads, rep, t = _run(net, 16, pool, feats, params, images, labels)
    except _sn().SchedulingError:
        pytest.skip("the reference schedule itself runs out of pool here")
    assert _bitwise(grads, base)


def test_graph_eager_and_parity_copies_are_bit_identical(cuda, alex32_case):
    net, params, images, labels = alex32_case
    _, base, _, _ = _run(net, 16, 1 << 30, ALL, params, images, labels, use_graph=True)
    _, eager, _, _ = _run(net, 16, 1 << 30, ALL, params, images, labels, use_graph=False)
    _, parity, _, t = _run(net, 16, 1 << 30, ALL, params, images, labels, elide_backups=False)
    assert t.d2h_bytes == 10822272  # every scheduled copy-out really issued (reference: 10,822,272 B)
    assert _bitwise(eager, base) and _bitwise(parity, base)


def test_alexnet_cache_knee_evictions_and_demand_fetches(cuda):
    """AlexNet b250 in a 1536 MiB pool with the LRU cache: the reference
    schedule evicts and demand-fetches 477,024,000 bytes; results must equal
    the roomy unscheduled run bit for bit."""
    from paper_1801_04380_b200.training import init_parameters
    net = _fixture("alexnet")
    params = init_parameters(net, seed=3, head_scale=0.1)
    images, labels = _inputs(net, 250, seed=5)
    _, base, _, _ = _run(net, 250, 8 << 30, "none", params, images, labels)
    loss, grads, rep, t = _run(net, 250, 1536 << 20, "cache", params, images, labels)
    assert rep.demand_transfer_bytes == 477024000 and rep.evictions > 0
    assert t.h2d_bytes == rep.demand_transfer_bytes + rep.scheduled_transfer_bytes - t.d2h_bytes or t.h2d_bytes > 0
    assert _bitwise(grads, base)


def test_resnet50g_small_batch_matches_oracle(cuda):
    from paper_1801_04380_b200.netgen import gen_resnet
    from paper_1801_04380_b200.training import init_parameters
    from oracle.numerics import forward_backward, relative_error
    net = gen_resnet(3, 4, 6, 3)
    params = init_parameters(net, seed=2, head_scale=0.1)
    images, labels = _inputs(net, 8)
    loss, grads, rep, _ = _run(net, 8, 4 << 30, ALL, params, images, labels)
    _, base, _, _ = _run(net, 8, 4 << 30, "none", params, images, labels)
    assert _bitwise(grads, base)
    ref_loss, _ = forward_backward(net, params, images, labels)
    assert abs(loss - ref_loss) <= 5e-3 * abs(ref_loss)
    ref, sens = _sensitivity(net, params, images, labels)
    worst = max(relative_error(grads[l][k], ref[l][k]) for l in ref for k in ("w", "b"))
    assert worst <= 3 * sens + 5e-3, (worst, sens)


def test_sgd_training_reduces_loss(cuda, alex32_case):
    sn = _sn()
    from paper_1801_04380_b200.training import Executor
    net, params, images, labels = alex32_case
    cfg = sn.SimConfig(pool_bytes=1 << 30, features=sn.parse_features(ALL), cost=sn.CostConfig(batch=16))
    ex = Executor(net, cfg, params=params, lr=0.005)
    ex.set_inputs(images, labels)
    losses = [ex.step(update=True)[0] for _ in range(40)]
    ex.close()
    assert min(losses[-5:]) < 0.8 * losses[0], losses


def test_layer_fusions_are_bit_identical(cuda, monkeypatch):
    """BN+ReLU forward/backward fusion (mask recomputed from the BN input), the
    elided BN output and the two-way JOIN backward give exactly the unfused
    one-kernel-per-layer results (SN_FUSE=0)."""
    from paper_1801_04380_b200.netgen import gen_resnet
    from paper_1801_04380_b200.training import init_parameters
    net = gen_resnet(1, 1, 2, 1)
    params = init_parameters(net, seed=6, head_scale=0.1)
    images, labels = _inputs(net, 4, seed=3)
    # the CONV-epilogue BN statistics and the BN-backward CONV bias gradient
    # sum in a different order (checked separately below); this test pins the
    # bit-exact fusions
    monkeypatch.setenv("SN_FUSE_REASSOC", "0")
    for feats in ("none", ALL):
        loss, grads, _, t = _run(net, 4, 4 << 30, feats, params, images, labels)
        monkeypatch.setenv("SN_FUSE", "0")
        loss0, grads0, _, t0 = _run(net, 4, 4 << 30, feats, params, images, labels)
        monkeypatch.delenv("SN_FUSE")
        assert t.kernels < t0.kernels
        assert loss == loss0 and _bitwise(grads, grads0)


def test_reassociating_fusions(cuda, monkeypatch):
    """BN statistics combined from the CONV epilogue's per-tile partials
    (shifted sums per 128-row tile, fp64 combination) and the CONV bias
    gradient summed in the BN backward's dx pass match the separate reduction
    passes to rounding.  On a smooth net (no ReLU / max-pool masks that a
    last-bit change can flip); a last-bit change of a BN output can still move
    its tf32 rounding in the next CONV (1 tf32 ulp = 2^-11 relative), so:
    loss rel. 1e-4, weight / BN gradients rel. 2e-3 (a wrong statistic or bias
    sum is off by O(1)); CONV biases (analytically zero before a BN, so pure
    rounding noise) abs. 2e-3 of the largest weight gradient.  The fused run is deterministic
    (bit-identical on repeat), also on ResNet-50g-style blocks."""
    from paper_1801_04380_b200.netgen import gen_resnet
    from paper_1801_04380_b200.training import init_parameters
    from oracle.numerics import relative_error
    sn = _sn()
    rnet = gen_resnet(1, 1, 2, 1)
    rparams = init_parameters(rnet, seed=6, head_scale=0.1)
    rimages, rlabels = _inputs(rnet, 8, seed=4)
    loss, grads, _, _ = _run(rnet, 8, 4 << 30, ALL, rparams, rimages, rlabels)
    loss_b, grads_b, _, _ = _run(rnet, 8, 4 << 30, ALL, rparams, rimages, rlabels)
    assert loss == loss_b and _bitwise(grads, grads_b)

    net = sn.parse_network(SMOOTH32, "smooth32")
    params = init_parameters(net, seed=3, head_scale=0.1)
    images, labels = _inputs(net, 8, seed=5)
    loss, grads, _, t = _run(net, 8, 1 << 30, ALL, params, images, labels)
    monkeypatch.setenv("SN_FUSE_REASSOC", "0")
    loss0, grads0, _, t0 = _run(net, 8, 1 << 30, ALL, params, images, labels)
    # (SMOOTH32's first CONV is the stem, whose weight gradient sums its own
    # bias gradient in both modes: the BN-side bias fusion saves no launch here)
    assert t.kernels <= t0.kernels
    assert abs(loss - loss0) <= 1e-4 * abs(loss0)
    kinds = {l.id: l.kind.name for l in net.layers}
    worst = max(relative_error(grads[l]["w"], grads0[l]["w"]) for l in grads)
    assert worst <= 2e-3, worst
    scale = max(float(grads0[l]["w"].abs().max()) for l in grads)
    for l in grads:
        if kinds[l] == "CONV" and kinds[net.layers[l].next[0]] == "BN":
            assert float((grads[l]["b"] - grads0[l]["b"]).abs().max()) <= 2e-3 * scale, net.layers[l].name
        else:
            assert relative_error(grads[l]["b"], grads0[l]["b"]) <= 2e-3, net.layers[l].name


@pytest.mark.parametrize("kind", ["densenet", "inception"])
def test_branchy_nets_match_oracle_and_are_schedule_invariant(cuda, kind):
    """Benchmark configs 3-4 (reduced): the DenseNet-121-style (k-way JOIN-sum,
    avg-pool transitions) and Inception-v4-style (4-branch modules, 3x3/s1 avg
    pools, 8x8 global pool) graphs execute under every scheduling feature with
    bit-identical gradients, and match the CPU oracle within the tf32
    tolerance of the other nets."""
    from paper_1801_04380_b200 import netgen
    from paper_1801_04380_b200.training import init_parameters
    from oracle.numerics import forward_backward, relative_error
    if kind == "densenet":
        net = netgen.gen_densenet(blocks=(2, 3, 2, 2), widths=(32, 64, 64, 64))
        batch = 4
    else:
        net = netgen.gen_inception(n_a=1, n_b=1, n_c=1)
        batch = 2
    params = init_parameters(net, seed=4, head_scale=0.1)
    images, labels = _inputs(net, batch, seed=7)
    loss, grads, rep, _ = _run(net, batch, 8 << 30, ALL, params, images, labels)
    for feats in ("none", "liveness,offload,recompute=memory"):
        l2, g2, _, _ = _run(net, batch, 8 << 30, feats, params, images, labels)
        assert l2 == loss and _bitwise(g2, grads), feats
    ref_loss, _ = forward_backward(net, params, images, labels)
    assert abs(loss - ref_loss) <= 5e-3 * abs(ref_loss), (loss, ref_loss)
    ref, sens = _sensitivity(net, params, images, labels)
    worst = max(relative_error(grads[l][k], ref[l][k]) for l in ref for k in ("w", "b"))
    assert worst <= 3 * sens + 5e-3, (worst, sens)


@pytest.mark.parametrize("feats", ["none", "liveness,offload,recompute=memory", ALL])
def test_dense_join_chain_backward_is_bit_identical(cuda, monkeypatch, feats):
    """DenseNet-style blocks: the nested JOIN-sum backwards run as one running
    sum (each JOIN adds its dy once and writes the inputs it finishes) instead
    of adding dy into every input's buffer -- same additions in the same order,
    so the same bits as the per-input JOIN backward (SN_FUSE_DENSE=0), with
    fewer launches when a chain applies."""
    from paper_1801_04380_b200 import netgen
    from paper_1801_04380_b200.training import init_parameters
    net = netgen.gen_densenet(blocks=(3, 10, 4, 2), widths=(32, 32, 64, 64))
    params = init_parameters(net, seed=8, head_scale=0.1)
    images, labels = _inputs(net, 4, seed=9)
    loss, grads, _, t = _run(net, 4, 8 << 30, feats, params, images, labels)
    monkeypatch.setenv("SN_FUSE_DENSE", "0")
    loss0, grads0, _, t0 = _run(net, 4, 8 << 30, feats, params, images, labels)
    assert loss == loss0 and _bitwise(grads, grads0)
    assert t.kernels < t0.kernels, (t.kernels, t0.kernels)


def test_pipelined_host_steps_match_serial_host_steps(cuda, alex32_case):
    """The prefetching end-to-end call (sn_exec_step_host_pipelined) trains
    exactly like one synchronous sn_exec_step_host per batch."""
    sn = _sn()
    from paper_1801_04380_b200.training import Executor
    net, params, _, _ = alex32_case
    batches = []
    for s in range(4):
        img, lab = _inputs(net, 16, seed=10 + 2 * s)
        batches.append((img.permute(0, 2, 3, 1).contiguous().pin_memory(), lab.to(torch.int32).pin_memory()))
    batches = batches + batches[:2]  # revisit buffers, like a loader's ring
    cfg = sn.SimConfig(pool_bytes=1 << 30, features=sn.parse_features(ALL), cost=sn.CostConfig(batch=16))
    runs = []
    for mode in ("serial", "loop", "pipelined"):
        ex = Executor(net, cfg, params=params, lr=0.005)
        if mode == "loop":  # sn_exec_train_host: one native call, losses read behind the next step
            losses = [l for l, _ in ex.train_host(batches)]
        elif mode == "pipelined":  # one sn_exec_step_host_pipelined call per step
            losses = [ex.step_host_pipelined(img, lab, *(batches[i + 1] if i + 1 < len(batches) else (None, None)))[0]
                      for i, (img, lab) in enumerate(batches)]
        else:
            losses = [ex.step_host(img, lab)[0] for img, lab in batches]
        runs.append((losses, ex.get("params")))
        ex.close()
    for r in runs[1:]:
        assert r[0] == runs[0][0]
        assert _bitwise(r[1], runs[0][1])


def test_wgrad_partials_use_the_planned_workspace(cuda, alex32_case):
    """With convselect the planner grants each CONV step a workspace (factor x
    output bytes from the free pool); the weight-gradient split-K partials live
    there, inside the pool, whenever they fit -- and the gradients stay
    bit-identical to a run without workspaces (the split count is per layer)."""
    sn = _sn()
    from paper_1801_04380_b200.training import Executor
    net, params, images, labels = alex32_case
    uses, grads = [], []
    for feats in ("liveness", "liveness,convselect"):
        cfg = sn.SimConfig(pool_bytes=1 << 30, features=sn.parse_features(feats), cost=sn.CostConfig(batch=16))
        ex = Executor(net, cfg, params=params)
        ex.set_inputs(images, labels)
        ex.step(update=False)
        uses.append(ex.workspace_use())
        grads.append(ex.get("grads"))
        ex.close()
    n_conv = sum(1 for l in net.layers if l.kind.name == "CONV")
    assert sum(uses[1]) == n_conv and uses[1][0] >= 1, uses
    assert _bitwise(grads[0], grads[1])


@pytest.mark.parametrize("graph", [True, False])
def test_transfer_stats_eager_and_graph(cuda, graph):
    """The copy-engine / exposed-fetch timers work in both execution modes
    (graph: external event-record nodes; eager: plain records): AlexNet b250 in
    a 1536 MiB cache pool fetches 477,024,000 bytes back on demand."""
    sn = _sn()
    from paper_1801_04380_b200.training import Executor, init_parameters
    net = _fixture("alexnet")
    params = init_parameters(net, seed=3, head_scale=0.1)
    images, labels = _inputs(net, 250, seed=5)
    cfg = sn.SimConfig(pool_bytes=1536 << 20, features=sn.parse_features("cache"), cost=sn.CostConfig(batch=250))
    ex = Executor(net, cfg, params=params, use_graph=graph)
    ex.set_inputs(images, labels)
    ex.step(update=False)
    ts = ex.transfer_stats()
    ex.close()
    assert ts["h2d_bytes"] >= 477024000 and ts["h2d_ms"] > 0 and ts["h2d_GBps"] > 1
    assert ts["d2h_bytes"] > 0 and ts["d2h_ms"] > 0
    assert ts["exposed_ms"] >= 0


# ---- fp32-faithful mode (precision="fp32": 3xTF32 split operands) ----------
# Stated tolerance: loss rel. err <= 1e-5 and every parameter gradient within
# 1e-4 relative Frobenius of the CPU fp32 oracle, masks included (fp32-level
# products leave only ~1e-6 activation differences, so ReLU / max-pool flips
# are rare single elements).  A CONV bias feeding a training-mode BN has an
# exactly-zero true gradient; it is compared absolutely against the layer's
# weight-gradient norm.
FP32_TOL = 1e-4


def _fp32_errors(net, grads, ref):
    sn = _sn()
    from oracle.numerics import relative_error
    errs = {}
    for l in ref:
        lay = net.layers[l]
        bn_fed = lay.kind is sn.LayerKind.CONV and any(net.layers[n].kind is sn.LayerKind.BN for n in lay.next)
        errs[(lay.name, "w")] = relative_error(grads[l]["w"], ref[l]["w"])
        if bn_fed:
            errs[(lay.name, "b")] = (grads[l]["b"] - ref[l]["b"]).norm().item() / ref[l]["w"].norm().item()
        else:
            errs[(lay.name, "b")] = relative_error(grads[l]["b"], ref[l]["b"])
    return errs


def _fp32_case(net, batch, pool, params, images, labels):
    from oracle.numerics import forward_backward
    loss, grads, rep, _ = _run(net, batch, pool, ALL, params, images, labels, precision="fp32")
    ref_loss, ref = forward_backward(net, params, images, labels)
    assert abs(loss - ref_loss) <= 1e-5 * abs(ref_loss), (loss, ref_loss)
    errs = _fp32_errors(net, grads, ref)
    assert max(errs.values()) <= FP32_TOL, sorted(errs.items(), key=lambda kv: -kv[1])[:4]
    return rep


def test_fp32_mode_smooth32_matches_oracle(cuda):
    from paper_1801_04380_b200.training import init_parameters
    net = _sn().parse_network(SMOOTH32, name="smooth32")
    params = init_parameters(net, seed=4, head_scale=0.1)
    images, labels = _inputs(net, 16)
    _fp32_case(net, 16, 1 << 30, params, images, labels)


def test_fp32_mode_alex32_matches_oracle(cuda, alex32_case):
    net, params, images, labels = alex32_case
    rep = _fp32_case(net, 16, 1 << 30, params, images, labels)
    assert rep.peak_bytes == 16777216


def test_fp32_mode_resnet50g_b8_matches_oracle(cuda):
    """ResNet-50g at batch 8 is ill-conditioned for any fp32 computation: the
    CPU fp32 oracle itself differs from the fp64 oracle by up to ~1e-2 on some
    BN / CONV gradients (training-mode BN over 8 x 7 x 7 values, 17 residual
    blocks).  Stated tolerance: every gradient of the fp32 mode is at least as
    close to the fp64 oracle as the CPU fp32 oracle is (within 2x), and within
    1e-4 wherever the CPU fp32 result is within 5e-6 of fp64; loss <= 1e-5."""
    import torch
    from oracle.numerics import forward_backward
    from paper_1801_04380_b200.netgen import gen_resnet
    from paper_1801_04380_b200.training import init_parameters
    net = gen_resnet(3, 4, 6, 3)
    params = init_parameters(net, seed=2, head_scale=0.1)
    images, labels = _inputs(net, 8)
    loss, grads, _, _ = _run(net, 8, 4 << 30, ALL, params, images, labels, precision="fp32")
    ref_loss, ref64 = forward_backward(net, params, images, labels, dtype=torch.float64)
    _, ref32 = forward_backward(net, params, images, labels)
    assert abs(loss - ref_loss) <= 1e-5 * abs(ref_loss), (loss, ref_loss)
    e_gpu = _fp32_errors(net, grads, ref64)
    e_cpu = _fp32_errors(net, ref32, ref64)
    bad = {k: (e_gpu[k], e_cpu[k]) for k in e_gpu
           if e_gpu[k] > max(2 * e_cpu[k], FP32_TOL if e_cpu[k] <= 5e-6 else 0.0) and e_gpu[k] > 5e-6}
    assert not bad, sorted(bad.items(), key=lambda kv: -kv[1][0])[:6]


def test_fp32_mode_feature_sets_are_bit_identical(cuda, alex32_case):
    net, params, images, labels = alex32_case
    base_loss, base, _, _ = _run(net, 16, 1 << 30, "none", params, images, labels, precision="fp32")
    loss, grads, _, _ = _run(net, 16, 17 << 20, ALL, params, images, labels, precision="fp32")
    assert loss == base_loss and _bitwise(grads, base)


# ---- data-parallel program path (NCCL communicator inside the executor) ----

@pytest.mark.parametrize("which", ["alex32", "resnet50g_b8"])
def test_dp_world1_nccl_path_is_bit_identical(cuda, alex32_case, which):
    """A world-size-1 NCCL communicator exercises the whole DP program path
    (bucketed ncclAllReduce on the communication stream after each bucket's
    backward steps, per-bucket fused SGD, stream joins, graph capture): after
    two update steps the parameters and gradients equal the single-replica
    executor's bit for bit."""
    sn = _sn()
    from paper_1801_04380_b200 import dp
    from paper_1801_04380_b200.training import Executor, init_parameters
    if which == "alex32":
        net, params, images, labels = alex32_case
        batch, pool = 16, 1 << 30
    else:
        from paper_1801_04380_b200.netgen import gen_resnet
        net = gen_resnet(3, 4, 6, 3)
        params = init_parameters(net, seed=2, head_scale=0.1)
        images, labels = _inputs(net, 8)
        batch, pool = 8, 4 << 30
    cfg = sn.SimConfig(pool_bytes=pool, features=sn.parse_features(ALL), cost=sn.CostConfig(batch=batch))
    out = []
    for use_dp in (False, True):
        ctx = dp.DPContext(force_comm=True) if use_dp else None
        ex = Executor(net, cfg, params=params, lr=0.01, dp=ctx, dp_bucket_bytes=1 << 20)
        ex.set_inputs(images, labels)
        losses = [ex.step(update=True)[0] for _ in range(2)]
        out.append((losses, ex.get("params"), ex.get("grads")))
        ex.close()
        if ctx:
            ctx.close()
    (l0, p0, g0), (l1, p1, g1) = out
    assert l0 == l1
    assert _bitwise(p0, p1) and _bitwise(g0, g1)
    assert any(not torch.equal(p0[l]['w'], params[l]['w']) for l in params)  # the updates ran


# ---- UTP backing store in device memory (peer HBM; loopback on one GPU) ----

def test_device_stash_loopback_is_bit_identical(cuda):
    """The Unified Tensor Pool's copy-out store in HBM (stash="device": an
    NVLink peer's memory, here the same GPU as a loopback) instead of pinned
    host memory: the AlexNet b250 cache-knee schedule (evictions and demand
    fetches of 477,024,000 bytes) gives bit-identical gradients, and the
    copies run device-to-device."""
    from paper_1801_04380_b200.training import init_parameters
    net = _fixture("alexnet")
    params = init_parameters(net, seed=3, head_scale=0.1)
    images, labels = _inputs(net, 250, seed=5)
    _, base, _, _ = _run(net, 250, 8 << 30, "none", params, images, labels)
    sn = _sn()
    from paper_1801_04380_b200.training import Executor
    cfg = sn.SimConfig(pool_bytes=1536 << 20, features=sn.parse_features("cache"), cost=sn.CostConfig(batch=250))
    ex = Executor(net, cfg, params=params, stash="device")
    ex.set_inputs(images, labels)
    _, t = ex.step(update=False)
    grads = ex.get("grads")
    mem = ex.memory()
    xfer = ex.transfer_stats()
    ex.close()
    assert _bitwise(grads, base)
    assert t.h2d_bytes > 0 and mem["device_stash_bytes"] > 0 and mem["host_stash_bytes"] == 0
    assert xfer["h2d_GBps"] and xfer["h2d_GBps"] > 100  # not PCIe-bound


def test_device_stash_parity_copies_bit_identical(cuda, alex32_case):
    net, params, images, labels = alex32_case
    _, base, _, _ = _run(net, 16, 1 << 30, ALL, params, images, labels)
    _, dev, _, t = _run(net, 16, 1 << 30, ALL, params, images, labels, elide_backups=False, stash="device")
    assert t.d2h_bytes == 10822272 and _bitwise(dev, base)


# ---- measured kernel-variant catalog (non-parity mode) ----------------------

def test_autotune_catalog_measures_and_trains(cuda):
    """autotune=True benchmarks every CONV kernel variant per layer shape and op
    at create time and runs the fastest (a non-parity mode: summation orders
    differ from the default variants).  The catalog covers every distinct
    shape x op with exactly one chosen variant, the chosen one is the fastest
    measured, and the step still matches the CPU oracle at the tf32
    tolerance."""
    from oracle.numerics import forward_backward, relative_error
    from paper_1801_04380_b200.netgen import gen_resnet
    from paper_1801_04380_b200.training import init_parameters
    net = gen_resnet(1, 1, 2, 1)
    params = init_parameters(net, seed=6, head_scale=0.1)
    images, labels = _inputs(net, 8, seed=3)
    sn = _sn()
    from paper_1801_04380_b200.training import Executor
    cfg = sn.SimConfig(pool_bytes=4 << 30, features=sn.parse_features(ALL), cost=sn.CostConfig(batch=8))
    ex = Executor(net, cfg, params=params, autotune=True)
    cat = ex.catalog()
    ex.set_inputs(images, labels)
    loss, _ = ex.step(update=False)
    grads = ex.get("grads")
    ex.close()
    assert cat and all(c["us"] > 0 for c in cat)
    groups = {}
    for c in cat:
        groups.setdefault((c["layer"], c["op"]), []).append(c)
    assert {op for _, op in groups} == {"fwd", "dgrad", "wgrad"}
    for g in groups.values():
        assert sum(c["chosen"] for c in g) == 1
        assert min(g, key=lambda c: c["us"])["chosen"]
    ref_loss, ref = forward_backward(net, params, images, labels)
    _, emu = forward_backward(net, params, images, labels, tf32=True)
    sens = max(relative_error(emu[l][k], ref[l][k]) for l in ref for k in ("w", "b"))
    worst = max(relative_error(grads[l][k], ref[l][k]) for l in ref for k in ("w", "b"))
    assert abs(loss - ref_loss) <= 5e-3 * abs(ref_loss)
    assert worst <= 3 * sens + 5e-3, (worst, sens)


def test_stem_bn_dx_fused_into_stem_wgrad_is_bit_identical(cuda, monkeypatch):
    """The stem BN's dx pass folded into the stem weight gradient (dx formed
    from the BN input and dy inside the kernel, never written) equals the
    materialised path bit for bit, with every other fusion on, and launches
    one kernel fewer; gathering dy from the stem max pool's gradient and
    argmax (the pool backward dropped) saves one more, same bits."""
    from paper_1801_04380_b200.netgen import gen_resnet
    from paper_1801_04380_b200.training import init_parameters
    net = gen_resnet(3, 4, 6, 3)
    params = init_parameters(net, seed=2, head_scale=0.1)
    images, labels = _inputs(net, 8)
    loss, grads, _, t = _run(net, 8, 4 << 30, ALL, params, images, labels)
    monkeypatch.setenv("SN_FUSE_POOL_GATHER", "0")
    loss1, grads1, _, t1 = _run(net, 8, 4 << 30, ALL, params, images, labels)
    monkeypatch.setenv("SN_FUSE_STEM_BN", "0")
    loss0, grads0, _, t0 = _run(net, 8, 4 << 30, ALL, params, images, labels)
    assert t1.kernels == t0.kernels - 1
    assert loss1 == loss0 and _bitwise(grads1, grads0)
    # and the stem pool backward gathered into both (the pool's dx never written)
    assert t.kernels == t1.kernels - 1
    assert loss == loss1 and _bitwise(grads, grads1)


@pytest.mark.parametrize("feats", ["liveness", "liveness,recompute=memory", "liveness,offload,cache"])
def test_stem_pool_gather_bit_identical_across_schedules(cuda, monkeypatch, feats):
    """The pool-ordered stem BN statistics give the same bits whether dy is
    gathered (pool backward dropped) or read from the materialised pool dx,
    under schedules that allow the gather and schedules that do not."""
    from paper_1801_04380_b200.netgen import gen_resnet
    from paper_1801_04380_b200.training import init_parameters
    net = gen_resnet(3, 4, 6, 3)
    params = init_parameters(net, seed=5, head_scale=0.1)
    images, labels = _inputs(net, 8)
    loss, grads, _, _ = _run(net, 8, 4 << 30, feats, params, images, labels)
    monkeypatch.setenv("SN_FUSE_POOL_GATHER", "0")
    loss0, grads0, _, _ = _run(net, 8, 4 << 30, feats, params, images, labels)
    assert loss == loss0 and _bitwise(grads, grads0)


@pytest.mark.parametrize("feats", ["none", ALL])
def test_batched_dgrad_weight_prep_is_bit_identical(cuda, monkeypatch, feats):
    """Every CONV's dgrad weight transform run once per step in one batched
    launch on the side stream (SN_DGRAD_PREP=1; the default for nets with >= 64
    such layers) gives exactly the per-dgrad transforms: flipped / transposed
    stride-1 filters and the sub-pixel blocks of the stride-2 convolutions."""
    from paper_1801_04380_b200.netgen import gen_resnet
    from paper_1801_04380_b200.training import init_parameters
    net = gen_resnet(1, 2, 2, 1)
    params = init_parameters(net, seed=8, head_scale=0.1)
    images, labels = _inputs(net, 4, seed=5)
    monkeypatch.setenv("SN_DGRAD_PREP", "1")
    loss1, grads1, _, t1 = _run(net, 4, 4 << 30, feats, params, images, labels)
    monkeypatch.setenv("SN_DGRAD_PREP", "0")
    loss0, grads0, _, t0 = _run(net, 4, 4 << 30, feats, params, images, labels)
    assert t1.kernels < t0.kernels  # one batched launch replaces one per layer
    assert loss1 == loss0 and _bitwise(grads1, grads0)


@pytest.mark.parametrize("feats", [ALL, "liveness,offload,recompute=memory"])
def test_bn_relu_fusion_over_a_freed_bn_input_is_bit_identical(cuda, monkeypatch, feats):
    """DenseNet-style layers: the JOIN output feeding BN -> ReLU is dropped right
    after the BN (recompute), before the ReLU runs; the fused BN apply at the
    ReLU still reads it -- planned only when nothing is allocated over it in
    between except the ReLU's own output at exactly its blocks (elementwise in
    place), and the dead-replay analysis keeps the replays it reads.  Bit-
    identical to one kernel per layer (SN_FUSE=0), with fewer kernels."""
    from paper_1801_04380_b200 import netgen
    from paper_1801_04380_b200.training import init_parameters
    net = netgen.gen_densenet(blocks=(3, 3, 2, 2), widths=(32, 64, 64, 64))
    params = init_parameters(net, seed=9, head_scale=0.1)
    images, labels = _inputs(net, 4, seed=2)
    monkeypatch.setenv("SN_FUSE_REASSOC", "0")
    loss, grads, _, t = _run(net, 4, 8 << 30, feats, params, images, labels)
    monkeypatch.setenv("SN_FUSE", "0")
    loss0, grads0, _, t0 = _run(net, 4, 8 << 30, feats, params, images, labels)
    assert t.kernels < t0.kernels
    assert loss == loss0 and _bitwise(grads, grads0)
