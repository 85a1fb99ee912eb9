"""Kernel-level accounting of one training iteration (measurement helpers for
bench.py and tools/launch_table.py; no effect on the training path).

* ``kernel_table(ex)``: every kernel of one iteration in issue order -- its
  tape action, layer, mangled name (``Executor.census``) and its CUDA-event time
  from a node-by-node replay of the iteration (``Executor.kernel_times``) --
  with the SURVEY 8(d) algorithmic GEMM FLOPs attributed to the tensor kernels
  (a CONV / FC action's forward, weight-gradient and data-gradient FLOPs split
  over the tcgen05 kernels that do that part).
"""

from __future__ import annotations

import math
import re

TYPES = ["fwd", "replay", "bwd", "other"]


def is_tensor(name: str) -> bool:
    return any(t in name for t in ("tc_conv", "tc_gemm", "stem_rows_kernel", "stem_wgrad_rows"))


def is_wgrad(name: str) -> bool:
    """Mangled names: the halo / stem weight-gradient kernels say so;
    tc_conv_tma_kernel<BN, STAGES, MODE, CG> is a weight gradient at MODE 1 or 3;
    tc_gemm_kernel<BN, STAGES, A_MN, B_MN, ...> with both operands MN-major."""
    if "wgrad" in name:
        return True
    if "tc_conv_tma_kernel" in name:
        ints = re.findall(r"Li(\d+)E", name.split("tc_conv_tma_kernel", 1)[1])
        return len(ints) >= 3 and ints[2] in ("1", "3")
    if "tc_gemm_kernel" in name:
        flags = re.findall(r"Lb([01])E", name.split("tc_gemm_kernel", 1)[1])
        return len(flags) >= 2 and flags[0] == "1" and flags[1] == "1"
    return False


def gemm_dims(net, shapes, lid: int, batch: int) -> dict:
    """Implicit-GEMM view of a CONV / FC layer: forward, wgrad and dgrad M x N x K."""
    lay = net.layers[lid]
    o, i = shapes[lid], shapes[lay.prev[0]]
    if lay.kind.value == "CONV":
        k = lay.params["k"]
        return {"fwd": (batch * o[1] * o[2], o[0], k * k * i[0]), "wgrad": (k * k * i[0], o[0], batch * o[1] * o[2]),
                "dgrad": (batch * i[1] * i[2], i[0], k * k * o[0])}
    fan = math.prod(i)
    return {"fwd": (batch, o[0], fan), "wgrad": (fan, o[0], batch), "dgrad": (batch, fan, o[0])}


def attribute_flops(actions: list[dict]) -> None:
    """Per kernel: ``flops`` and ``part`` for the tensor kernels of CONV / FC
    actions (actions: {"type", "gemm" (optional), "kernels": [{"name", ...}]})."""
    for a in actions:
        tk = [k for k in a["kernels"] if is_tensor(k["name"])]
        for k in a["kernels"]:
            k["flops"], k["part"] = 0.0, ""
        if "gemm" not in a or not tk:
            continue
        if a["type"] == "bwd":
            groups = {"wgrad": [k for k in tk if is_wgrad(k["name"])],
                      "dgrad": [k for k in tk if not is_wgrad(k["name"])]}
        else:
            groups = {"fwd": tk}
        for part, ks in groups.items():
            M, N, K = a["gemm"][part]
            for k in ks:
                k["flops"], k["part"] = 2.0 * M * N * K / len(ks), part


def kernel_table(ex, reps: int = 3) -> list[dict]:
    """Actions of one iteration with their kernels, event-timed and attributed."""
    from .costmodel import propagate_shapes
    net = ex.net
    shapes = propagate_shapes(net)
    census = ex.census()
    prof = ex.profile()
    times = ex.kernel_times(reps)
    actions = []
    it = iter(times)
    for i, (names, (_, lid, typ)) in enumerate(zip(census, prof)):
        a = {"i": i, "layer": lid, "type": TYPES[typ], "kernels": []}
        for nm in names:
            act, us = next(it)
            assert act == i, "kernel replay out of step with the census"
            a["kernels"].append({"name": nm, "us": us})
        if lid >= 0:
            lay = net.layers[lid]
            a["name"], a["kind"] = lay.name, lay.kind.value
            if lay.kind.value in ("CONV", "FC"):
                a["gemm"] = gemm_dims(net, shapes, lid, ex.batch)
        actions.append(a)
    attribute_flops(actions)
    return actions
