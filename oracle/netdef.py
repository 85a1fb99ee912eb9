"""ORACLE (test infrastructure only) -- network text, shapes, layer constants
and parameter initialisation, restated independently of the product package.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module.  Nothing here imports ``paper_1801_04380_b200``:
the oracle reads the reference's ``.net`` text itself, so a wrong constant or
shape rule in the product cannot also hide in its checker.

Restated from the reference (memsched 0.1.0, /root/reference/pkg/src/memsched):
  * ``.net`` text: ``layer <name> <KIND> [k=v ...]`` / ``edge <src> <dst>`` /
    ``#`` comments; values coerced int -> float -> str (netgraph.py:160-169,
    :172-233).  Layer ids follow declaration order; ``prev`` / ``next`` follow
    edge order.  (Validation errors are the product's business; the oracle
    only needs well-formed nets.)
  * shapes: CONV/POOL windows ``(h + 2p - k) // s + 1`` with POOL stride
    defaulting to k and CONV stride to 1; FC -> (out,); everything else keeps
    its input shape (costmodel.py:113-155).
  * the residual generator ``gen_resnet`` (netgen.py:51-109): stem 7x7/2 CONV,
    BN, ACT, 3x3/2 POOL; per block one 3x3 CONV+BN+ACT, JOIN-sum skips except
    on the stride-2 first block of stages 2-4; a 7x7 POOL, FC, SOFTMAX.

Numeric semantics the reference leaves open (it has no tensors),
as this repo states them (README of the executor):
  POOL  ``mode=max`` (padding never wins) or ``mode=avg`` (divisor k*k, padding
        counted); LRN ``size=5 alpha=1e-4 beta=0.75 k=2.0`` unless given,
        y = x / (k + alpha/size * sum_window x^2)^beta; DROPOUT ``rate=0.5``
        unless given; BN batch statistics, ``eps=1e-5``; SOFTMAX terminal with
        mean cross-entropy; ACT = ReLU; JOIN = elementwise sum; FC flattens
        its input in (h, w, c) order.
  Parameters: He-uniform CONV / FC weights (bound sqrt(6 / fan_in), fan_in =
  k*k*Cin or the flattened input), biases uniform in +-1/sqrt(fan_in), drawn
  weight-then-bias in layer-id order from one CPU generator; BN gamma 1,
  beta 0; CONV weights KRSC, FC weights [out][in].
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

KINDS = ("DATA", "CONV", "POOL", "ACT", "LRN", "BN", "FC", "DROPOUT", "SOFTMAX", "JOIN")


@dataclass
class OLayer:
    id: int
    name: str
    kind: str
    params: dict
    prev: list = field(default_factory=list)
    next: list = field(default_factory=list)


@dataclass
class ONet:
    name: str
    layers: list

    @property
    def data_id(self) -> int:
        return next(l.id for l in self.layers if l.kind == "DATA" and not l.prev)

    @property
    def terminal_id(self) -> int:
        return next(l.id for l in self.layers if l.kind == "SOFTMAX")


def _value(text: str):
    for conv in (int, float):
        try:
            return conv(text)
        except ValueError:
            pass
    return text


def parse_net(text: str, name: str = "net") -> ONet:
    layers: list[OLayer] = []
    ids: dict[str, int] = {}
    for raw in text.splitlines():
        toks = raw.split("#", 1)[0].split()
        if not toks:
            continue
        if toks[0] == "layer":
            params = {}
            for kv in toks[3:]:
                k, _, v = kv.partition("=")
                params[k] = _value(v)
            if toks[2] not in KINDS:
                raise ValueError(f"oracle: unknown layer kind {toks[2]!r}")
            ids[toks[1]] = len(layers)
            layers.append(OLayer(len(layers), toks[1], toks[2], params))
        elif toks[0] == "edge":
            a, b = ids[toks[1]], ids[toks[2]]
            layers[a].next.append(b)
            layers[b].prev.append(a)
        else:
            raise ValueError(f"oracle: unknown directive {toks[0]!r}")
    return ONet(name, layers)


def as_onet(net) -> ONet:
    """``.net`` text, an ONet, or any object with ``.layers`` whose items carry
    ``name``, ``kind`` (an enum with ``.value`` / ``.name``, or a string),
    ``params``, ``prev``, ``next`` -- the data is copied, no code is called."""
    if isinstance(net, ONet):
        return net
    if isinstance(net, str):
        return parse_net(net)
    out = []
    for i, l in enumerate(net.layers):
        kind = l.kind if isinstance(l.kind, str) else getattr(l.kind, "value", None) or l.kind.name
        out.append(OLayer(i, str(l.name), str(kind), dict(l.params), list(l.prev), list(l.next)))
    return ONet(str(getattr(net, "name", "net")), out)


def topo_order(net: ONet) -> list[int]:
    """Any topological order gives the same numbers (each layer is a function of
    its inputs); Kahn's algorithm, lowest id first."""
    pending = [len(l.prev) for l in net.layers]
    ready = sorted(l.id for l in net.layers if not l.prev)
    order = []
    while ready:
        lid = ready.pop(0)
        order.append(lid)
        for n in net.layers[lid].next:
            pending[n] -= 1
            if pending[n] == 0:
                ready.append(n)
        ready.sort()
    if len(order) != len(net.layers):
        raise ValueError("oracle: cyclic or unreachable layers")
    return order


def _window(x: int, k: int, s: int, p: int) -> int:
    return (x + 2 * p - k) // s + 1


def shapes(net: ONet) -> dict[int, tuple[int, ...]]:
    out: dict[int, tuple[int, ...]] = {}
    for lid in topo_order(net):
        l = net.layers[lid]
        p = l.params
        if l.kind == "DATA":
            out[lid] = (int(p["c"]), int(p["h"]), int(p["w"]))
            continue
        src = out[l.prev[0]]
        if l.kind == "CONV":
            k, s, pd = int(p["k"]), int(p.get("s", 1)), int(p.get("p", 0))
            out[lid] = (int(p["out"]), _window(src[1], k, s, pd), _window(src[2], k, s, pd))
        elif l.kind == "POOL":
            k = int(p["k"])
            s, pd = int(p.get("s", k)), int(p.get("p", 0))
            out[lid] = (src[0], _window(src[1], k, s, pd), _window(src[2], k, s, pd))
        elif l.kind == "FC":
            out[lid] = (int(p["out"]),)
        else:
            out[lid] = src
    return out


@dataclass(frozen=True)
class Consts:
    pool_avg: bool
    lrn_size: int
    lrn_alpha: float
    lrn_beta: float
    lrn_k: float
    dropout_rate: float
    bn_eps: float


def _num(p: dict, key: str, default):
    v = p.get(key, default)
    return v if isinstance(v, (int, float)) and not isinstance(v, bool) else default


def constants(layer: OLayer) -> Consts:
    p = layer.params
    mode = p.get("mode", "max")
    if mode not in ("max", "avg"):
        raise ValueError(f"oracle: POOL mode {mode!r}")
    return Consts(pool_avg=mode == "avg", lrn_size=int(_num(p, "size", 5)), lrn_alpha=float(_num(p, "alpha", 1e-4)),
                  lrn_beta=float(_num(p, "beta", 0.75)), lrn_k=float(_num(p, "k", 2.0)) if layer.kind == "LRN" else 2.0,
                  dropout_rate=float(_num(p, "rate", 0.5)), bn_eps=float(_num(p, "eps", 1e-5)))


def init_parameters(net, seed: int = 2, head_scale: float = 1.0) -> dict[int, dict]:
    import torch
    net = as_onet(net)
    shp = shapes(net)
    g = torch.Generator().manual_seed(seed)
    head = set(net.layers[net.terminal_id].prev)
    params: dict[int, dict] = {}
    for l in net.layers:
        if l.kind == "BN":
            c = shp[l.id][0]
            params[l.id] = {"w": torch.ones(c), "b": torch.zeros(c)}
            continue
        if l.kind == "CONV":
            k = int(l.params["k"])
            wshape = (shp[l.id][0], k, k, shp[l.prev[0]][0])
        elif l.kind == "FC":
            wshape = (shp[l.id][0], math.prod(shp[l.prev[0]]))
        else:
            continue
        fan_in = math.prod(wshape[1:])
        w = (torch.rand(wshape, generator=g) * 2 - 1) * math.sqrt(6.0 / fan_in)
        b = (torch.rand((wshape[0],), generator=g) * 2 - 1) / math.sqrt(fan_in)
        if l.id in head:
            w, b = w * head_scale, b * head_scale
        params[l.id] = {"w": w, "b": b}
    return params


def resnet_text(n1: int, n2: int, n3: int, n4: int, num_classes: int = 1000) -> str:
    """The reference's generated residual net (avg classifier pooling)."""
    L: list[str] = ["layer data DATA c=3 h=224 w=224", "layer conv_stem CONV out=64 k=7 s=2 p=3",
                    "layer bn_stem BN", "layer relu_stem ACT", "layer pool_stem POOL k=3 s=2 p=1",
                    "edge data conv_stem", "edge conv_stem bn_stem", "edge bn_stem relu_stem",
                    "edge relu_stem pool_stem"]
    trunk = "pool_stem"
    for stage, blocks in enumerate((n1, n2, n3, n4), start=1):
        for b in range(1, blocks + 1):
            tag = f"s{stage}b{b}"
            down = stage > 1 and b == 1
            L += [f"layer conv_{tag} CONV out={64 << (stage - 1)} k=3 s={2 if down else 1} p=1",
                  f"layer bn_{tag} BN", f"layer relu_{tag} ACT",
                  f"edge {trunk} conv_{tag}", f"edge conv_{tag} bn_{tag}", f"edge bn_{tag} relu_{tag}"]
            if down:
                trunk = f"relu_{tag}"
            else:
                L += [f"layer join_{tag} JOIN", f"edge relu_{tag} join_{tag}", f"edge {trunk} join_{tag}"]
                trunk = f"join_{tag}"
    L += ["layer pool_avg POOL k=7 s=1 mode=avg", f"layer fc FC out={num_classes}", "layer softmax SOFTMAX",
          f"edge {trunk} pool_avg", "edge pool_avg fc", "edge fc softmax"]
    return "\n".join(L) + "\n"


def conv_fc_flops(net, batch: int) -> dict[int, tuple[int, int]]:
    """Algorithmic tensor FLOPs per iteration and layer: (forward,
    backward) with backward = wgrad + dgrad (dgrad omitted when the input is DATA)."""
    net = as_onet(net)
    shp = shapes(net)
    out = {}
    for l in net.layers:
        if l.kind not in ("CONV", "FC"):
            continue
        o, i = shp[l.id], shp[l.prev[0]]
        if l.kind == "CONV":
            k = int(l.params["k"])
            mac = batch * o[0] * o[1] * o[2] * i[0] * k * k
        else:
            mac = batch * o[0] * math.prod(i)
        dgrad = net.layers[l.prev[0]].kind != "DATA"
        out[l.id] = (2 * mac, 2 * mac * (2 if dgrad else 1))
    return out
