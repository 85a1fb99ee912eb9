"""Per-layer byte and time costs (drop-in for memsched costmodel.py).

The arithmetic runs in the C++ planner (``csrc/planner/core.cpp``,
``build_costs``), which is also what the executor and scheduler use, so the
numbers a caller inspects are by construction the ones the schedule and the
B200 arena are built from.  Byte counts are exact: ``batch * prod(shape) *
dtype_bytes``; DATA occupies no device bytes; parameters are accounted
outside the pool; ACT/DROPOUT gradients alias their producer's buffer.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _cabi
from .errors import CostError
from .netgraph import GRAD_INPLACE_KINDS, LayerKind, NetworkDef

__all__ = ["CostConfig", "LayerCost", "CostError", "HEAVY_KINDS", "build_costs",
           "propagate_shapes", "grad_owner", "baseline_peak_bytes", "total_forward_bytes",
           "total_grad_bytes", "mib"]

HEAVY_KINDS = frozenset({LayerKind.CONV, LayerKind.FC})


@dataclass(frozen=True)
class CostConfig:
    """Cost-model knobs (reference costmodel.py:32-51; same defaults)."""

    batch: int = 200
    dtype_bytes: int = 4
    time_per_elem: float = 2e-9
    heavy_time_per_elem: float = 2e-8
    backward_time_factor: float = 2.0
    bandwidth_bytes_per_s: float = 8e9

    def __post_init__(self) -> None:
        checks = (
            (self.batch < 1, f"batch must be positive, got {self.batch}"),
            (self.dtype_bytes < 1, "dtype_bytes must be positive"),
            (self.bandwidth_bytes_per_s <= 0, "bandwidth must be positive"),
            (self.backward_time_factor <= 0, "backward_time_factor must be positive"),
        )
        for bad, msg in checks:
            if bad:
                raise CostError(msg)


@dataclass(frozen=True)
class LayerCost:
    layer_id: int
    shape: tuple[int, ...]
    out_elems: int
    out_bytes: int
    device_bytes: int
    grad_bytes: int
    param_bytes: int
    fwd_time: float
    bwd_time: float


CostTable = dict[int, LayerCost]


def _planner_config(cfg: CostConfig):
    from .simulator import Features
    return _cabi.sim_config(1, Features(), cfg)


def _cost_rows(net: NetworkDef, cfg: CostConfig):
    handle = _cabi.PlanHandle(net, _planner_config(cfg), mode="costs")
    return handle.costs()


def build_costs(net: NetworkDef, config: CostConfig) -> CostTable:
    table: CostTable = {}
    for lid, c in enumerate(_cost_rows(net, config)):
        table[lid] = LayerCost(
            layer_id=lid, shape=tuple(c.shape[: c.ndim]), out_elems=c.out_elems,
            out_bytes=c.out_bytes, device_bytes=c.device_bytes, grad_bytes=c.grad_bytes,
            param_bytes=c.param_bytes, fwd_time=c.fwd_time, bwd_time=c.bwd_time)
    return table


def propagate_shapes(net: NetworkDef) -> dict[int, tuple[int, ...]]:
    """Per-sample output shape of every layer."""
    rows = _cost_rows(net, CostConfig(batch=1))
    return {lid: tuple(c.shape[: c.ndim]) for lid, c in enumerate(rows)}


def grad_owner(net: NetworkDef, layer_id: int) -> int | None:
    """The layer whose gradient buffer holds d(output of ``layer_id``)."""
    lid = layer_id
    while net.layers[lid].kind in GRAD_INPLACE_KINDS:
        lid = net.layers[lid].prev[0]
    return None if net.layers[lid].kind is LayerKind.DATA else lid


def total_forward_bytes(costs: CostTable) -> int:
    return sum(c.device_bytes for c in costs.values())


def total_grad_bytes(costs: CostTable) -> int:
    return sum(c.grad_bytes for c in costs.values())


def baseline_peak_bytes(costs: CostTable) -> int:
    """Bytes held at the end of an iteration with every feature off."""
    return total_forward_bytes(costs) + total_grad_bytes(costs)


def mib(nbytes: int | float) -> float:
    return nbytes / (1 << 20)
