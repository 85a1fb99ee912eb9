"""Scheduler entry points: ``run_simulation`` / ``run_sweep`` (drop-in API).

Same types and semantics as memsched simulator.py:45-170, 734-783.  The
decisions -- residency ledger, block-pool offsets, LRU eviction, transfers,
replays, workspace selection -- are made by the C++ planner
(``libsnplan.so``), bit-identical to the reference (tests/test_sched_parity.py
checks every SimReport field, row, selection and the full event tape against
golden vectors produced by the reference itself).  ``run_training``
(``training.py``) executes the same plan on a B200.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

from . import _cabi
from .convselect import Selection
from .costmodel import CostConfig
from .errors import ConfigError
from .netgraph import NetworkDef

__all__ = ["Features", "parse_features", "SimConfig", "StepRow", "SimReport", "SweepPoint",
           "FEATURE_NAMES", "SWEEP_AXES", "POLICIES", "run_simulation", "run_sweep", "plan_handle"]

FEATURE_NAMES = ("liveness", "offload", "cache", "recompute", "convselect")
POLICIES = ("speed", "memory", "cost-aware")
SWEEP_AXES = ("batch", "pool-bytes")
_PHASES = ("forward", "backward", "replay")


@dataclass(frozen=True)
class Features:
    liveness: bool = False
    offload: bool = False
    cache: bool = False
    recompute: str | None = None
    convselect: bool = False

    def normalized(self) -> "Features":
        """cache implies offload; offload or recompute imply liveness."""
        offload = self.offload or self.cache
        liveness = self.liveness or offload or bool(self.recompute)
        return replace(self, liveness=liveness, offload=offload)

    def label(self) -> str:
        parts = [n for n in ("liveness", "offload", "cache") if getattr(self, n)]
        if self.recompute:
            parts.append(f"recompute={self.recompute}")
        if self.convselect:
            parts.append("convselect")
        return ",".join(parts) or "none"


def parse_features(text: str) -> Features:
    """``liveness,offload,cache,recompute[=speed|memory|cost-aware],convselect``."""
    text = text.strip()
    if text in ("", "none"):
        return Features()
    chosen: dict[str, object] = {}
    for token in (t.strip() for t in text.split(",")):
        if not token:
            continue
        name, eq, value = token.partition("=")
        if name not in FEATURE_NAMES:
            raise ConfigError(f"unknown feature {name!r}, expected one of {FEATURE_NAMES}")
        if name == "recompute":
            policy = value if eq else "cost-aware"
            if policy not in POLICIES:
                raise ConfigError(f"unknown recompute policy {policy!r}, expected one of {POLICIES}")
            chosen[name] = policy
        elif eq:
            raise ConfigError(f"feature {name!r} takes no value")
        else:
            chosen[name] = True
    return Features(**chosen)


@dataclass(frozen=True)
class SimConfig:
    pool_bytes: int
    features: Features = Features()
    cost: CostConfig = CostConfig()

    def __post_init__(self) -> None:
        if self.pool_bytes <= 0:
            raise ConfigError(f"pool size must be positive, got {self.pool_bytes}")


@dataclass(frozen=True)
class StepRow:
    index: float
    layer: str
    kind: str
    phase: str
    resident_bytes: int
    live_count: int
    pool_used_bytes: int
    compute_s: float
    stall_s: float
    transfer_bytes: int


@dataclass(frozen=True)
class SimReport:
    net_name: str
    num_layers: int
    num_steps: int
    batch: int
    pool_capacity_bytes: int
    features: str
    recompute_policy: str | None
    recompute_modes: tuple[str, ...]
    peak_bytes: int
    peak_step: int
    peak_layer: str
    peak_live_count: int
    peak_working_bytes: int
    peak_stash_bytes: int
    min_pool_bytes: int
    baseline_peak_bytes: int
    liveness_peak_bytes: int
    compute_s: float
    stall_s: float
    stall_prefetch_s: float
    stall_demand_s: float
    stall_backup_s: float
    transfer_busy_s: float
    total_s: float
    scheduled_transfer_bytes: int
    scheduled_transfer_count: int
    demand_transfer_bytes: int
    demand_transfer_count: int
    cache_hits: int
    evictions: int
    extra_forward_steps: int
    planned_extra_forward_steps: int
    pool_high_water_bytes: int
    selections: tuple[Selection, ...]
    rows: tuple[StepRow, ...]


def plan_handle(net: NetworkDef, config: SimConfig) -> "_cabi.PlanHandle":
    """Plan one iteration in the native planner (raises the reference errors)."""
    return _cabi.PlanHandle(net, _cabi.sim_config(config.pool_bytes, config.features, config.cost))


def report_from_handle(net: NetworkDef, config: SimConfig, h: "_cabi.PlanHandle") -> SimReport:
    r = h.report()
    feats = config.features.normalized()
    names = [l.name for l in net.layers]
    kinds = [l.kind.value for l in net.layers]
    rows = tuple(
        StepRow(index=x.index, layer=names[x.layer], kind=kinds[x.layer], phase=_PHASES[x.phase],
                resident_bytes=x.resident_bytes, live_count=x.live_count,
                pool_used_bytes=x.pool_used_bytes, compute_s=x.compute_s, stall_s=x.stall_s,
                transfer_bytes=x.transfer_bytes)
        for x in h.rows())
    sels = tuple(
        Selection(step=s.step, layer_id=s.layer, layer_name=names[s.layer],
                  phase=_PHASES[s.phase], algo=_cabi.ALGO_NAMES[s.algo],
                  workspace_bytes=s.workspace_bytes, free_bytes=s.free_bytes)
        for s in h.selections())
    modes = tuple(_cabi.RC_NAME[m] for m in h.modes()) if feats.recompute else ()
    return SimReport(
        net_name=net.name, num_layers=r.num_layers, num_steps=r.num_steps,
        batch=config.cost.batch, pool_capacity_bytes=config.pool_bytes, features=feats.label(),
        recompute_policy=feats.recompute, recompute_modes=modes, peak_bytes=r.peak_bytes,
        peak_step=r.peak_step, peak_layer=names[r.peak_layer], peak_live_count=r.peak_live_count,
        peak_working_bytes=r.peak_working_bytes, peak_stash_bytes=r.peak_stash_bytes,
        min_pool_bytes=r.min_pool_bytes, baseline_peak_bytes=r.baseline_peak_bytes,
        liveness_peak_bytes=r.liveness_peak_bytes, compute_s=r.compute_s, stall_s=r.stall_s,
        stall_prefetch_s=r.stall_prefetch_s, stall_demand_s=r.stall_demand_s,
        stall_backup_s=r.stall_backup_s, transfer_busy_s=r.transfer_busy_s, total_s=r.total_s,
        scheduled_transfer_bytes=r.scheduled_transfer_bytes,
        scheduled_transfer_count=r.scheduled_transfer_count,
        demand_transfer_bytes=r.demand_transfer_bytes,
        demand_transfer_count=r.demand_transfer_count, cache_hits=r.cache_hits,
        evictions=r.evictions, extra_forward_steps=r.extra_forward_steps,
        planned_extra_forward_steps=r.planned_extra_forward_steps,
        pool_high_water_bytes=r.pool_high_water_bytes, selections=sels, rows=rows)


def run_simulation(net: NetworkDef, config: SimConfig) -> SimReport:
    return report_from_handle(net, config, plan_handle(net, config))


@dataclass(frozen=True)
class SweepPoint:
    axis: str
    value: int
    peak_bytes: int
    peak_step: int
    total_s: float
    compute_s: float
    stall_s: float
    scheduled_transfer_bytes: int
    demand_transfer_bytes: int
    extra_forward_steps: int
    pool_high_water_bytes: int


def run_sweep(net: NetworkDef, config: SimConfig, axis: str, values: list[int]) -> list[SweepPoint]:
    if axis not in SWEEP_AXES:
        raise ConfigError(f"unknown sweep axis {axis!r}, expected one of {SWEEP_AXES}")
    if not values:
        raise ConfigError("sweep needs at least one value")
    out: list[SweepPoint] = []
    for value in values:
        if axis == "batch":
            cfg = replace(config, cost=replace(config.cost, batch=value))
        else:
            cfg = replace(config, pool_bytes=value)
        rep = run_simulation(net, cfg)
        out.append(SweepPoint(
            axis=axis, value=value, peak_bytes=rep.peak_bytes, peak_step=rep.peak_step,
            total_s=rep.total_s, compute_s=rep.compute_s, stall_s=rep.stall_s,
            scheduled_transfer_bytes=rep.scheduled_transfer_bytes,
            demand_transfer_bytes=rep.demand_transfer_bytes,
            extra_forward_steps=rep.extra_forward_steps,
            pool_high_water_bytes=rep.pool_high_water_bytes))
    return out
