"""Static analyses of the reference API: liveness, offload plan, recompute plan.

Drop-in for memsched ``liveness.py``, ``offload.py`` and ``recompute.py``
(same names, same results -- pinned by tests/test_analysis_parity.py against
golden vectors from the reference).  The planner computes the same quantities
in C++ (``csrc/planner/analysis.cpp``) for the simulation; these Python
entry points serve callers that inspect them directly.  Where the planner
already has the answer (``step_demands``), it is fetched from it.

Tables are built once per call in O(N) (the reference rebuilds the backward
use table once per segment).
"""

from __future__ import annotations

import io
from collections import OrderedDict
from dataclasses import dataclass

from . import _cabi
from .costmodel import CostConfig, CostTable, grad_owner
from .errors import AllLockedError, ConfigError
from .netgraph import (BACKWARD_NEEDS, OFFLOAD_KINDS, LayerKind, NetworkDef, Schedule, backward_reads,
                       checkpoint_segments, external_inputs)

__all__ = [
    "forward_use_steps", "backward_use_steps", "last_use_step", "last_forward_use_step", "GradBuffer",
    "grad_buffers", "TensorLife", "liveness_table", "dump_liveness_csv", "resident_curve", "curve_peak",
    "working_set_bytes", "liveness_peak", "offload_candidates", "OffloadPlan", "build_offload_plan", "LruCache",
    "AllLockedError", "POLICIES", "Segment", "RecomputePlan", "build_segments", "first_backward_use",
    "memory_extras", "speed_extras", "speed_prediction", "plan", "DemandPeak", "step_demands", "min_pool_bytes",
    "demand_peak",
]

# ---------------------------------------------------------------- liveness


def _use_table(net: NetworkDef, sched: Schedule, backward: bool) -> dict[int, list[int]]:
    uses: dict[int, list[int]] = {l.id: [] for l in net.layers}
    for lay in net.layers:
        if backward:
            step = sched.bwd_step_of[lay.id]
            for t in backward_reads(net, lay.id):
                uses[t].append(step)
        else:
            step = sched.fwd_step_of[lay.id]
            for p in lay.prev:
                uses[p].append(step)
    for v in uses.values():
        v.sort()
    return uses


def forward_use_steps(net: NetworkDef, sched: Schedule) -> dict[int, list[int]]:
    return _use_table(net, sched, backward=False)


def backward_use_steps(net: NetworkDef, sched: Schedule) -> dict[int, list[int]]:
    return _use_table(net, sched, backward=True)


def last_forward_use_step(net: NetworkDef, sched: Schedule) -> dict[int, int]:
    fwd = forward_use_steps(net, sched)
    return {lid: max([sched.fwd_step_of[lid], *steps]) for lid, steps in fwd.items()}


def last_use_step(net: NetworkDef, sched: Schedule) -> dict[int, int]:
    fwd = forward_use_steps(net, sched)
    bwd = backward_use_steps(net, sched)
    return {lid: max([sched.fwd_step_of[lid], *fwd[lid], *bwd[lid]]) for lid in fwd}


@dataclass(frozen=True)
class GradBuffer:
    owner: int
    nbytes: int
    create_step: int
    free_step: int


def grad_buffers(net: NetworkDef, costs: CostTable, sched: Schedule,
                 materialize_seed: bool = False) -> dict[int, GradBuffer]:
    """Gradient buffers keyed by owner (sorted), alive from the first writer's
    backward step to the owner's own backward step."""
    first: dict[int, int] = {}

    def note(owner, step):
        if owner is not None and (owner not in first or step < first[owner]):
            first[owner] = step

    for lay in net.layers:
        if lay.kind is LayerKind.DATA:
            continue
        for p in lay.prev:
            note(grad_owner(net, p), sched.bwd_step_of[lay.id])
    if materialize_seed:
        term = net.terminal_id
        note(grad_owner(net, term), sched.bwd_step_of[term])
    return {o: GradBuffer(o, costs[o].grad_bytes, first[o], sched.bwd_step_of[o]) for o in sorted(first)}


@dataclass(frozen=True)
class TensorLife:
    layer_id: int
    name: str
    kind: str
    nbytes: int
    birth_step: int
    last_forward_use: int
    last_use: int


def liveness_table(net: NetworkDef, costs: CostTable, sched: Schedule) -> list[TensorLife]:
    last = last_use_step(net, sched)
    last_fwd = last_forward_use_step(net, sched)
    return [TensorLife(lid, net.layers[lid].name, net.layers[lid].kind.value, costs[lid].device_bytes,
                       sched.fwd_step_of[lid], last_fwd[lid], last[lid]) for lid in sched.forward_ids]


def dump_liveness_csv(net: NetworkDef, costs: CostTable, sched: Schedule) -> str:
    buf = io.StringIO()
    buf.write("layer,kind,bytes,birth_step,last_forward_use,last_use\n")
    for r in liveness_table(net, costs, sched):
        buf.write(f"{r.name},{r.kind},{r.nbytes},{r.birth_step},{r.last_forward_use},{r.last_use}\n")
    return buf.getvalue()


def resident_curve(net: NetworkDef, costs: CostTable, sched: Schedule, mode: str = "liveness") -> list[int]:
    """Bytes resident at each step; ``baseline`` frees nothing and keeps the seed."""
    if mode not in ("liveness", "baseline"):
        raise ValueError(f"unknown residency mode {mode!r}")
    n_steps = sched.num_steps
    delta = [0] * (n_steps + 1)

    def span(lo, hi, nbytes):
        delta[lo] += nbytes
        delta[hi + 1] -= nbytes

    end = n_steps - 1
    last = last_use_step(net, sched)
    for lid in sched.forward_ids:
        nb = costs[lid].device_bytes
        if nb:
            span(sched.fwd_step_of[lid], last[lid] if mode == "liveness" else end, nb)
    for buf in grad_buffers(net, costs, sched, materialize_seed=(mode == "baseline")).values():
        if buf.nbytes:
            hi = buf.free_step if mode == "liveness" else end
            if buf.create_step <= hi:
                span(buf.create_step, hi, buf.nbytes)
    curve, run = [], 0
    for s in range(n_steps):
        run += delta[s]
        curve.append(run)
    return curve


def curve_peak(curve: list[int]) -> tuple[int, int]:
    peak = max(curve)
    return peak, curve.index(peak)


def working_set_bytes(net: NetworkDef, costs: CostTable, sched: Schedule, buffers: dict[int, GradBuffer],
                      step: int) -> int:
    lay = net.layers[sched.steps[step].layer_id]
    if step < len(sched.forward_ids):
        return costs[lay.id].device_bytes + sum(costs[p].device_bytes for p in lay.prev)
    total = sum(costs[t].device_bytes for t in dict.fromkeys(backward_reads(net, lay.id)))
    seen: set[int] = set()
    dy = grad_owner(net, lay.id)
    if dy is not None and dy in buffers and buffers[dy].create_step <= step <= buffers[dy].free_step:
        total += buffers[dy].nbytes
        seen.add(dy)
    for p in lay.prev:
        o = grad_owner(net, p)
        if o is not None and o not in seen and o in buffers:
            seen.add(o)
            total += buffers[o].nbytes
    return total


def liveness_peak(net: NetworkDef, costs: CostTable, sched: Schedule) -> tuple[int, int]:
    return curve_peak(resident_curve(net, costs, sched, mode="liveness"))


# ---------------------------------------------------------------- offload


def offload_candidates(net: NetworkDef, kinds: frozenset[LayerKind] = OFFLOAD_KINDS,
                       order: list[int] | None = None) -> list[int]:
    ids = order if order is not None else [l.id for l in net.layers]
    return [lid for lid in ids if net.layers[lid].kind in kinds]


@dataclass(frozen=True)
class OffloadPlan:
    cp_ids: tuple[int, ...]
    drop_after: dict[int, int]
    prefetch_issue: dict[int, int]
    first_backward_use: dict[int, int]
    last_backward_use: dict[int, int]


def build_offload_plan(net: NetworkDef, sched: Schedule, cp_ids: list[int] | None = None) -> OffloadPlan:
    """Copy out after the last forward use; fetch one checkpoint ahead, never
    later than the first backward use."""
    cps = offload_candidates(net, order=sched.forward_ids) if cp_ids is None else list(cp_ids)
    bwd = backward_use_steps(net, sched)
    last_fwd = last_forward_use_step(net, sched)
    drop, issue, first, last = {}, {}, {}, {}
    for pos, cp in enumerate(cps):
        drop[cp] = last_fwd[cp]
        uses = bwd[cp]
        if not uses:
            continue
        first[cp], last[cp] = uses[0], uses[-1]
        nxt = sched.bwd_step_of[cps[pos + 1]] if pos + 1 < len(cps) else uses[0]
        issue[cp] = min(nxt, uses[0])
    return OffloadPlan(tuple(cps), drop, issue, first, last)


class LruCache:
    """Recency-ordered registry of reusable device tensors (locks never taken
    by the scheduler itself, but supported)."""

    def __init__(self) -> None:
        self._order: OrderedDict[object, list[int]] = OrderedDict()  # key -> [nbytes, locks]

    def __contains__(self, key: object) -> bool:
        return key in self._order

    def __len__(self) -> int:
        return len(self._order)

    def insert(self, key: object, nbytes: int) -> None:
        if key in self._order:
            self._order.move_to_end(key)
        else:
            self._order[key] = [nbytes, 0]

    def touch(self, key: object) -> None:
        self._order.move_to_end(key)

    def lock(self, key: object) -> None:
        self._order[key][1] += 1

    def unlock(self, key: object) -> None:
        entry = self._order[key]
        if entry[1] <= 0:
            raise ValueError(f"cache entry {key!r} is not locked")
        entry[1] -= 1

    def discard(self, key: object) -> int:
        entry = self._order.pop(key, None)
        return entry[0] if entry else 0

    def evict_lru(self) -> tuple[object, int]:
        for key, (nbytes, locks) in self._order.items():
            if locks == 0:
                del self._order[key]
                return key, nbytes
        raise AllLockedError("no unlocked cached tensor is available for eviction")

    def keys(self) -> list[object]:
        return list(self._order)


# ---------------------------------------------------------------- recompute

POLICIES = ("speed", "memory", "cost-aware")


@dataclass(frozen=True)
class Segment:
    index: int
    members: tuple[int, ...]
    anchors: tuple[int, ...]


@dataclass(frozen=True)
class RecomputePlan:
    policy: str
    segments: tuple[Segment, ...]
    modes: tuple[str, ...]
    spill_ids: frozenset[int]
    extra_forward_steps: int
    predictions: tuple[int, ...]

    def segment_of(self, layer_id: int) -> int | None:
        return next((s.index for s in self.segments if layer_id in s.members), None)


def build_segments(net: NetworkDef, sched: Schedule) -> list[Segment]:
    return [Segment(i, tuple(run), tuple(external_inputs(net, run)))
            for i, run in enumerate(checkpoint_segments(net, order=sched.forward_ids))]


def first_backward_use(net: NetworkDef, sched: Schedule, seg: Segment, _uses=None) -> int | None:
    uses = _uses if _uses is not None else backward_use_steps(net, sched)
    steps = [s for m in seg.members for s in uses[m]]
    return min(steps) if steps else None


def memory_extras(net: NetworkDef, seg: Segment) -> int:
    return sum(i + 1 for i, m in enumerate(seg.members) if BACKWARD_NEEDS[net.layers[m].kind])


def speed_extras(net: NetworkDef, sched: Schedule, seg: Segment, _uses=None) -> int:
    return len(seg.members) if first_backward_use(net, sched, seg, _uses) is not None else 0


def speed_prediction(net: NetworkDef, costs: CostTable, sched: Schedule, seg: Segment, _uses=None) -> int:
    step = first_backward_use(net, sched, seg, _uses)
    if step is None:
        return 0
    total = sum(costs[a].device_bytes for a in seg.anchors) + sum(costs[m].device_bytes for m in seg.members)
    user = sched.steps[step].layer_id
    dy = grad_owner(net, user)
    if dy is not None and user != net.terminal_id:
        total += costs[dy].grad_bytes
    for p in net.layers[user].prev:
        o = grad_owner(net, p)
        if o is not None and o != dy:
            total += costs[o].grad_bytes
    return total


def plan(net: NetworkDef, costs: CostTable, sched: Schedule, policy: str,
         offloaded_ids: frozenset[int] = frozenset()) -> RecomputePlan:
    if policy not in POLICIES:
        raise ConfigError(f"unknown recompute policy {policy!r}, expected one of {POLICIES}")
    segments = build_segments(net, sched)
    uses = backward_use_steps(net, sched)
    preds = [speed_prediction(net, costs, sched, s, uses) for s in segments]
    if policy == "cost-aware":
        floor = min_pool_bytes(net, costs, sched)
        modes = ["speed" if preds[s.index] <= floor else "memory" for s in segments]
    else:
        modes = [policy] * len(segments)
    extras = sum(speed_extras(net, sched, s, uses) if m == "speed" else memory_extras(net, s)
                 for s, m in zip(segments, modes))
    members = {m for s in segments for m in s.members}
    spills: set[int] = set()
    for lay in net.layers:
        if lay.kind is LayerKind.DATA:
            continue
        spills.update(r for r in backward_reads(net, lay.id)
                      if r not in members and r not in offloaded_ids and costs[r].device_bytes > 0)
    for seg, mode in zip(segments, modes):
        spills.update(a for a in seg.anchors if a not in offloaded_ids and costs[a].device_bytes > 0)
        if mode == "memory":
            inside = set(seg.members)
            spills.update(m for m in seg.members if any(n not in inside for n in net.layers[m].next))
    return RecomputePlan(policy, tuple(segments), tuple(modes), frozenset(spills), extras, tuple(preds))


@dataclass(frozen=True)
class DemandPeak:
    nbytes: int
    step: int
    layer_id: int


def step_demands(net: NetworkDef, costs: CostTable, sched: Schedule) -> list[int]:
    """Per-step bytes under the memory strategy (the schedulable floor's terms),
    computed by the C++ planner (``analysis.cpp: step_demands``).

    The cost table fixes batch and dtype size (out_elems = batch * prod(shape),
    out_bytes = out_elems * dtype_bytes); the planner rebuilds the identical
    table from them.
    """
    import math

    from .simulator import Features
    c0 = costs[net.layers[0].id]
    batch = c0.out_elems // math.prod(c0.shape)
    dtype = c0.out_bytes // c0.out_elems
    cfg = _cabi.sim_config(1, Features(), CostConfig(batch=batch, dtype_bytes=dtype))
    return _cabi.PlanHandle(net, cfg, mode="analyze").demands()


def min_pool_bytes(net: NetworkDef, costs: CostTable, sched: Schedule) -> int:
    return max(step_demands(net, costs, sched))


def demand_peak(net: NetworkDef, costs: CostTable, sched: Schedule) -> DemandPeak:
    demands = step_demands(net, costs, sched)
    peak = max(demands)
    step = demands.index(peak)
    return DemandPeak(peak, step, sched.steps[step].layer_id)
