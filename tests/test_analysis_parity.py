"""Analysis entry points and the block allocator vs golden vectors from the
reference (tests/golden/analysis_golden.json.gz, tests/golden/make_golden.py):
use steps, last uses, gradient-buffer windows, liveness table/CSV, residency
curves, working sets, the offload plan, recompute segments/extras/predictions,
every recompute policy's plan, step demands (max_i(l_i)), and random
alloc/free traces through the C++ BlockPool (offsets, exhaustion messages,
used bytes and high water after every operation).
"""

from __future__ import annotations

import dataclasses
import gzip
import json
from pathlib import Path

import pytest

import paper_1801_04380_b200 as sn
from paper_1801_04380_b200 import analysis as an
from paper_1801_04380_b200.errors import PoolExhausted
from paper_1801_04380_b200.poolalloc import BlockPool

with gzip.open(Path(__file__).parent / "golden" / "analysis_golden.json.gz", "rt") as _fh:
    _G = json.load(_fh)

CASES = _G["analysis"]


def _keyed(d):
    return {str(k): v for k, v in d.items()}


@pytest.mark.parametrize("case", CASES, ids=[f"{c['name']}/b{c['batch']}" for c in CASES])
def test_analysis_matches_reference(case):
    net = sn.parse_network(case["text"], name=case["name"])
    costs = sn.build_costs(net, sn.CostConfig(batch=case["batch"]))
    sched = sn.build_schedule(net)
    assert sched.forward_ids == case["forward_ids"]
    got_costs = [[list(c.shape), c.out_elems, c.out_bytes, c.device_bytes, c.grad_bytes, c.param_bytes,
                  c.fwd_time, c.bwd_time] for c in costs.values()]
    assert got_costs == case["costs"]
    assert _keyed(an.forward_use_steps(net, sched)) == case["fwd_uses"]
    assert _keyed(an.backward_use_steps(net, sched)) == case["bwd_uses"]
    assert _keyed(an.last_use_step(net, sched)) == case["last_use"]
    assert _keyed(an.last_forward_use_step(net, sched)) == case["last_fwd_use"]
    for seed in (0, 1):
        got = [list(dataclasses.astuple(b)) for b in an.grad_buffers(net, costs, sched, bool(seed)).values()]
        assert got == case[f"grad_buffers_{seed}"]
    assert [list(dataclasses.astuple(r)) for r in an.liveness_table(net, costs, sched)] == case["liveness_table"]
    assert an.dump_liveness_csv(net, costs, sched) == case["liveness_csv"]
    assert an.resident_curve(net, costs, sched, "liveness") == case["curve_liveness"]
    assert an.resident_curve(net, costs, sched, "baseline") == case["curve_baseline"]
    assert list(an.liveness_peak(net, costs, sched)) == case["liveness_peak"]
    bufs = an.grad_buffers(net, costs, sched, False)
    assert [an.working_set_bytes(net, costs, sched, bufs, s) for s in range(sched.num_steps)] == case["working_set"]
    op = an.build_offload_plan(net, sched)
    assert [list(op.cp_ids), _keyed(op.drop_after), _keyed(op.prefetch_issue), _keyed(op.first_backward_use),
            _keyed(op.last_backward_use)] == case["offload_plan"]
    segs = an.build_segments(net, sched)
    got = [[s.index, list(s.members), list(s.anchors), an.first_backward_use(net, sched, s),
            an.memory_extras(net, s), an.speed_extras(net, sched, s), an.speed_prediction(net, costs, sched, s)]
           for s in segs]
    assert got == case["segments"]
    for key, want in case["plans"].items():
        pol, off = key.split("/")
        p = an.plan(net, costs, sched, pol, frozenset(op.cp_ids) if off == "1" else frozenset())
        assert [list(p.modes), sorted(p.spill_ids), p.extra_forward_steps, list(p.predictions)] == want, key
    assert an.step_demands(net, costs, sched) == case["step_demands"]
    dp = an.demand_peak(net, costs, sched)
    assert [dp.nbytes, dp.step, dp.layer_id] == case["demand_peak"]
    assert an.min_pool_bytes(net, costs, sched) == max(case["step_demands"])


@pytest.mark.parametrize("trace", _G["pool_traces"], ids=lambda t: f"seed{t['seed']}")
def test_block_pool_matches_reference_trace(trace):
    pool = BlockPool(trace["capacity_blocks"] * 1024)
    for op in trace["trace"]:
        if op[0] == "F":
            pool.free(op[1])
            continue
        _, key, nbytes, high, want, used, hw = op
        if isinstance(want, str):
            with pytest.raises(PoolExhausted) as info:
                pool.alloc(key, nbytes, high=bool(high))
            assert str(info.value) == want
        else:
            assert pool.alloc(key, nbytes, high=bool(high)) == want
        assert (pool.used_bytes, pool.high_water_bytes) == (used, hw)
    pool.check()


def test_lru_cache_semantics():
    c = an.LruCache()
    c.insert("a", 1)
    c.insert("b", 2)
    c.insert("a", 1)  # duplicate insert is a touch (reference offload.py:100-104)
    assert c.keys() == ["b", "a"]
    c.lock("b")
    assert c.evict_lru() == ("a", 1)
    with pytest.raises(sn.AllLockedError):
        c.evict_lru()
    c.unlock("b")
    assert c.evict_lru() == ("b", 2)
