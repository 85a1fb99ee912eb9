"""Network generators for the benchmark configurations.

``resnet_text`` / ``gen_resnet`` emit the reference's generated residual nets
(memsched netgen.py:51-109: one 3x3 CONV+BN+ACT per block, JOIN-sum skips,
stride-2 first block of stages 2-4), layer for layer and edge for edge, so
their schedules are the reference's.  The classifier pooling carries
``mode=avg`` (a parameter the cost model ignores, so the schedule is
unchanged) because the executor needs a pooling mode and global average
pooling is what a ResNet uses.

``make_uniform_chain`` is the reference's closed-form test chain and
``random_fanjoin`` its seeded fan-out/fan-in property-test generator
(memsched netgen.py:112-171): the same ``random.Random(seed)`` draws in the
same order, so a seed gives the reference's network text exactly.
``densenet_text`` / ``inception_text`` build the JOIN-sum DenseNet-121- and
Inception-v4-style graphs of benchmark configs 3-4 (the reference ships no
generator for them; the reference parser accepts their text unchanged).
"""

from __future__ import annotations

import random

from .errors import ConfigError
from .netgraph import NetworkDef, parse_network

__all__ = ["resnet_text", "gen_resnet", "uniform_chain_text", "make_uniform_chain",
           "fanjoin_text", "random_fanjoin",
           "densenet_text", "gen_densenet", "inception_text", "gen_inception"]


class _Text:
    """Accumulates ``layer``/``edge`` lines."""

    def __init__(self) -> None:
        self.lines: list[str] = []

    def layer(self, name: str, kind: str, **params) -> str:
        extra = "".join(f" {k}={v}" for k, v in params.items())
        self.lines.append(f"layer {name} {kind}{extra}")
        return name

    def edge(self, src: str, dst: str) -> None:
        self.lines.append(f"edge {src} {dst}")

    def text(self) -> str:
        return "\n".join(self.lines) + "\n"


def resnet_text(n1: int, n2: int, n3: int, n4: int, num_classes: int = 1000,
                avg_mode: bool = True) -> str:
    blocks = (n1, n2, n3, n4)
    if min(blocks) < 1:
        raise ConfigError("each stage needs at least one block")
    t = _Text()
    t.layer("data", "DATA", c=3, h=224, w=224)
    t.layer("conv_stem", "CONV", out=64, k=7, s=2, p=3)
    t.layer("bn_stem", "BN")
    t.layer("relu_stem", "ACT")
    t.layer("pool_stem", "POOL", k=3, s=2, p=1)
    for a, b in (("data", "conv_stem"), ("conv_stem", "bn_stem"), ("bn_stem", "relu_stem"),
                 ("relu_stem", "pool_stem")):
        t.edge(a, b)
    trunk = "pool_stem"
    for stage, count in enumerate(blocks, start=1):
        width = 64 << (stage - 1)
        for b in range(1, count + 1):
            tag = f"s{stage}b{b}"
            stride = 2 if (stage > 1 and b == 1) else 1
            conv = t.layer(f"conv_{tag}", "CONV", out=width, k=3, s=stride, p=1)
            bn = t.layer(f"bn_{tag}", "BN")
            act = t.layer(f"relu_{tag}", "ACT")
            t.edge(trunk, conv)
            t.edge(conv, bn)
            t.edge(bn, act)
            if stride == 1:
                join = t.layer(f"join_{tag}", "JOIN")
                t.edge(act, join)
                t.edge(trunk, join)
                trunk = join
            else:
                trunk = act
    if avg_mode:
        t.layer("pool_avg", "POOL", k=7, s=1, mode="avg")
    else:
        t.layer("pool_avg", "POOL", k=7, s=1)
    t.layer("fc", "FC", out=num_classes)
    t.layer("softmax", "SOFTMAX")
    t.edge(trunk, "pool_avg")
    t.edge("pool_avg", "fc")
    t.edge("fc", "softmax")
    return t.text()


def gen_resnet(n1: int, n2: int, n3: int, n4: int, num_classes: int = 1000,
               avg_mode: bool = True) -> NetworkDef:
    depth = 3 * (n1 + n2 + n3 + n4) + 2
    return parse_network(resnet_text(n1, n2, n3, n4, num_classes, avg_mode), name=f"resnet{depth}")


def uniform_chain_text(n_layers: int, cp_positions: tuple[int, ...] = (), c: int = 4, h: int = 16,
                       w: int = 16) -> str:
    """Shape-preserving chain: 1x1 CONVs at ``cp_positions`` (1-based), else LRN/BN."""
    if n_layers < 2:
        raise ConfigError("chain needs at least 2 layers")
    cps = set(cp_positions)
    out_of_range = [p for p in cps if not 1 <= p <= n_layers]
    if out_of_range:
        raise ConfigError(f"checkpoint positions out of range: {out_of_range}")
    t = _Text()
    t.layer("data", "DATA", c=c, h=h, w=w)
    for i in range(1, n_layers + 1):
        if i in cps:
            t.layer(f"l{i}", "CONV", out=c, k=1)
        else:
            t.layer(f"l{i}", "LRN" if i % 2 else "BN")
    t.edge("data", "l1")
    for i in range(1, n_layers):
        t.edge(f"l{i}", f"l{i + 1}")
    return t.text()


def make_uniform_chain(n_layers: int, cp_positions: tuple[int, ...] = (), c: int = 4, h: int = 16,
                       w: int = 16) -> NetworkDef:
    return parse_network(uniform_chain_text(n_layers, cp_positions, c, h, w), name=f"chain{n_layers}")


# Layer kinds a fan-join branch draws from (reference netgen.py:112).
FANJOIN_BRANCH_KINDS = ("ACT", "LRN", "BN", "CONV")


def fanjoin_text(seed: int, min_blocks: int = 2, max_blocks: int = 5) -> str:
    """Text of the seeded fan-out/fan-in net: a spine of blocks, each 2-3
    shape-preserving branches of 1-2 layers summed by a JOIN, a 2x2 POOL after
    a block with probability 0.4 while h >= 4, then FC + SOFTMAX.  Every layer
    line precedes every edge line, as in the reference."""
    rng = random.Random(seed)
    c = rng.choice((2, 3, 4))
    hw = rng.choice((8, 16))
    layers = [f"layer data DATA c={c} h={hw} w={hw}"]
    edges: list[str] = []
    counter = [0]

    def name(prefix: str) -> str:
        counter[0] += 1
        return f"{prefix}{counter[0]}"

    spine = "data"
    for _ in range(rng.randint(min_blocks, max_blocks)):
        tails = []
        for _ in range(rng.randint(2, 3)):
            at = spine
            for _ in range(rng.randint(1, 2)):
                kind = rng.choice(FANJOIN_BRANCH_KINDS)
                lname = name(kind.lower())
                if kind == "CONV":
                    k = rng.choice((1, 3))
                    layers.append(f"layer {lname} CONV out={c} k={k} p={1 if k == 3 else 0}")
                else:
                    layers.append(f"layer {lname} {kind}")
                edges.append(f"edge {at} {lname}")
                at = lname
            tails.append(at)
        join = name("join")
        layers.append(f"layer {join} JOIN")
        edges.extend(f"edge {t} {join}" for t in tails)
        spine = join
        if hw >= 4 and rng.random() < 0.4:
            pool = name("pool")
            layers.append(f"layer {pool} POOL k=2 s=2")
            edges.append(f"edge {spine} {pool}")
            spine = pool
            hw //= 2
    fc = name("fc")
    layers.append(f"layer {fc} FC out={rng.choice((10, 16, 32))}")
    edges.append(f"edge {spine} {fc}")
    sm = name("softmax")
    layers.append(f"layer {sm} SOFTMAX")
    edges.append(f"edge {fc} {sm}")
    return "\n".join(layers + edges) + "\n"


def random_fanjoin(seed: int, min_blocks: int = 2, max_blocks: int = 5) -> NetworkDef:
    return parse_network(fanjoin_text(seed, min_blocks, max_blocks), name=f"fanjoin_{seed}")


# ---------------------------------------------------------------------------
# Benchmark configs 3-4: JOIN-sum variants (the .net format has no concat).

def densenet_text(blocks: tuple[int, ...] = (6, 12, 24, 16), widths: tuple[int, ...] = (64, 128, 256, 512),
                  num_classes: int = 1000) -> str:
    """DenseNet-121-style: every layer of a block reads the JOIN-sum of the block
    input and all earlier layer outputs (dense connectivity with sum instead of
    concat); a layer is BN-ACT-CONV1x1-BN-ACT-CONV3x3; transitions are
    BN-ACT-CONV1x1-avgPOOL2."""
    t = _Text()
    t.layer("data", "DATA", c=3, h=224, w=224)
    t.layer("conv0", "CONV", out=widths[0], k=7, s=2, p=3)
    t.layer("bn0", "BN")
    t.layer("relu0", "ACT")
    t.layer("pool0", "POOL", k=3, s=2, p=1)
    for a, b in (("data", "conv0"), ("conv0", "bn0"), ("bn0", "relu0"), ("relu0", "pool0")):
        t.edge(a, b)
    block_in = "pool0"
    for bi, (count, width) in enumerate(zip(blocks, widths), start=1):
        feats = [block_in]
        for li in range(1, count + 1):
            tag = f"b{bi}l{li}"
            if len(feats) == 1:
                src = feats[0]
            else:
                src = t.layer(f"cat_{tag}", "JOIN")
                for f in feats:
                    t.edge(f, src)
            bn1 = t.layer(f"bn1_{tag}", "BN")
            r1 = t.layer(f"relu1_{tag}", "ACT")
            c1 = t.layer(f"conv1_{tag}", "CONV", out=width, k=1)
            bn2 = t.layer(f"bn2_{tag}", "BN")
            r2 = t.layer(f"relu2_{tag}", "ACT")
            c2 = t.layer(f"conv2_{tag}", "CONV", out=width, k=3, p=1)
            for a, b in ((src, bn1), (bn1, r1), (r1, c1), (c1, bn2), (bn2, r2), (r2, c2)):
                t.edge(a, b)
            feats.append(c2)
        out = t.layer(f"cat_b{bi}", "JOIN")
        for f in feats:
            t.edge(f, out)
        if bi < len(blocks):
            bn = t.layer(f"bn_t{bi}", "BN")
            r = t.layer(f"relu_t{bi}", "ACT")
            cv = t.layer(f"conv_t{bi}", "CONV", out=widths[bi], k=1)
            pl = t.layer(f"pool_t{bi}", "POOL", k=2, s=2, mode="avg")
            for a, b in ((out, bn), (bn, r), (r, cv), (cv, pl)):
                t.edge(a, b)
            block_in = pl
        else:
            block_in = out
    t.layer("bn_final", "BN")
    t.layer("relu_final", "ACT")
    t.layer("pool_avg", "POOL", k=7, s=1, mode="avg")
    t.layer("fc", "FC", out=num_classes)
    t.layer("softmax", "SOFTMAX")
    for a, b in ((block_in, "bn_final"), ("bn_final", "relu_final"), ("relu_final", "pool_avg"),
                 ("pool_avg", "fc"), ("fc", "softmax")):
        t.edge(a, b)
    return t.text()


def gen_densenet(**kw) -> NetworkDef:
    return parse_network(densenet_text(**kw), name="densenet121s")


def inception_text(n_a: int = 4, n_b: int = 7, n_c: int = 3, num_classes: int = 1000) -> str:
    """Inception-v4-style at 299x299: stem, then A/B/C modules whose 4 branches
    (1x1; 1x1-3x3; 1x1-3x3-3x3; avgpool-1x1) are merged by JOIN-sum, with
    stride-2 reduction convs between module groups."""
    t = _Text()
    t.layer("data", "DATA", c=3, h=299, w=299)
    stem = [("stem1", dict(out=32, k=3, s=2)), ("stem2", dict(out=32, k=3)),
            ("stem3", dict(out=64, k=3, p=1)), ("stem4", dict(out=96, k=3, s=2)),
            ("stem5", dict(out=192, k=3)), ("stem6", dict(out=384, k=3, s=2))]
    prev = "data"
    for name, params in stem:
        t.layer(f"conv_{name}", "CONV", **params)
        t.layer(f"bn_{name}", "BN")
        t.layer(f"relu_{name}", "ACT")
        t.edge(prev, f"conv_{name}")
        t.edge(f"conv_{name}", f"bn_{name}")
        t.edge(f"bn_{name}", f"relu_{name}")
        prev = f"relu_{name}"

    def unit(tag: str, src: str, out: int, k: int, s: int = 1) -> str:
        c = t.layer(f"conv_{tag}", "CONV", out=out, k=k, s=s, p=(k // 2 if s == 1 else 0))
        b = t.layer(f"bn_{tag}", "BN")
        r = t.layer(f"relu_{tag}", "ACT")
        t.edge(src, c)
        t.edge(c, b)
        t.edge(b, r)
        return r

    def module(tag: str, src: str, width: int) -> str:
        heads = [unit(f"{tag}_1x1", src, width, 1)]
        heads.append(unit(f"{tag}_b2b", unit(f"{tag}_b2a", src, width // 2, 1), width, 3))
        x = unit(f"{tag}_b3a", src, width // 2, 1)
        x = unit(f"{tag}_b3b", x, width, 3)
        heads.append(unit(f"{tag}_b3c", x, width, 3))
        pool = t.layer(f"pool_{tag}", "POOL", k=3, s=1, p=1, mode="avg")
        t.edge(src, pool)
        heads.append(unit(f"{tag}_b4", pool, width, 1))
        join = t.layer(f"join_{tag}", "JOIN")
        for h in heads:
            t.edge(h, join)
        return join

    x = prev
    for group, (count, width) in enumerate(((n_a, 384), (n_b, 768), (n_c, 1536))):
        for i in range(count):
            x = module(f"{'abc'[group]}{i + 1}", x, width)
        if group < 2:
            x = unit(f"red{group + 1}", x, (768, 1536)[group], 3, s=2)
    t.layer("pool_avg", "POOL", k=8, s=1, mode="avg")
    t.layer("fc", "FC", out=num_classes)
    t.layer("softmax", "SOFTMAX")
    t.edge(x, "pool_avg")
    t.edge("pool_avg", "fc")
    t.edge("fc", "softmax")
    return t.text()


def gen_inception(**kw) -> NetworkDef:
    return parse_network(inception_text(**kw), name="inception4s")
