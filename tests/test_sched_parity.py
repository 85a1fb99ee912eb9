"""Schedule parity: the C++ planner against golden vectors from the reference.

tests/golden/sched_golden.json.gz was produced by tests/golden/make_golden.py
running the reference simulator (memsched 0.1.0) itself;
tests/golden/sched_golden_branchy.json.gz (make_golden.py --branchy) holds the
Inception-v4-style and DenseNet-121-style graphs of benchmark configs 3-4.  For every case the
planner must reproduce, bit for bit: every SimReport field (integers and IEEE
doubles), every StepRow, every Selection, the recompute modes, and the full
physical event tape (block offsets of every alloc, frees, copies, fetches,
replays, LRU operations, compute points) -- or raise the same exception type
with the same message.
"""

from __future__ import annotations

import dataclasses
import gzip
import hashlib
import json
from pathlib import Path

import pytest

import paper_1801_04380_b200 as sn
from paper_1801_04380_b200 import simulator as snsim

GOLDEN = Path(__file__).parent / "golden" / "sched_golden.json.gz"
GOLDEN_BRANCHY = Path(__file__).parent / "golden" / "sched_golden_branchy.json.gz"


def _load(path):
    with gzip.open(path, "rt") as fh:
        return json.load(fh)


_DATA = _load(GOLDEN)
_BRANCHY = _load(GOLDEN_BRANCHY)
_NETS = {**_DATA["nets"], **_BRANCHY["nets"]}
_CASES = _DATA["cases"]
_BRANCHY_CASES = _BRANCHY["cases"]


def canon(obj) -> str:
    return json.dumps(obj, separators=(",", ":"))


def digest(obj) -> str:
    return hashlib.sha256(canon(obj).encode()).hexdigest()


def _net(case):
    return sn.parse_network(_NETS[case["net"]], name=case["name"])


def _config(case):
    return sn.SimConfig(pool_bytes=case["pool"], features=sn.parse_features(case["features"]),
                        cost=sn.CostConfig(batch=case["batch"], **case.get("cost", {})))


def _run(case):
    net = _net(case)
    cfg = _config(case)
    h = snsim.plan_handle(net, cfg)
    return snsim.report_from_handle(net, cfg, h), h


def _report_dict(rep):
    out = {}
    for f in dataclasses.fields(rep):
        v = getattr(rep, f.name)
        if f.name == "rows":
            v = [list(dataclasses.astuple(r)) for r in v]
        elif f.name == "selections":
            v = [list(dataclasses.astuple(s)) for s in v]
        elif f.name == "recompute_modes":
            v = list(v)
        out[f.name] = v
    return out


def _ids(cases):
    return [c["id"] for c in cases]


def check_case(case):
    if "error" in case:
        with pytest.raises(Exception) as info:
            _run(case)
        exc = info.value
        assert type(exc).__name__ == case["error"][0], (type(exc), str(exc))
        assert str(exc) == case["error"][1]
        return
    rep, h = _run(case)
    got = _report_dict(rep)
    rows, sels = got.pop("rows"), got.pop("selections")
    want = case["report"]
    for key, val in want.items():
        assert got[key] == val and type(got[key]) is type(val), (key, got[key], val)
    if "rows" in case:
        assert rows == case["rows"]
    assert digest(rows) == case["rows_sha"]
    if "selections" in case:
        assert sels == case["selections"]
    assert digest(sels) == case["sel_sha"]
    tape = h.tape_as_lists()
    if "tape" in case:
        for i, (a, b) in enumerate(zip(tape, case["tape"])):
            assert a == b, f"tape diverges at event {i}: got {a}, want {b}"
        assert len(tape) == len(case["tape"])
    assert len(tape) == case["tape_len"]
    assert digest(tape) == case["tape_sha"]


_SMALL = [c for c in _CASES if not c["id"].startswith(("resnet2534", "resnet830", "resnet842"))]
_DEEP = [c for c in _CASES if c["id"].startswith(("resnet2534", "resnet830", "resnet842"))]


@pytest.mark.parametrize("case", _SMALL, ids=_ids(_SMALL))
def test_schedule_matches_reference(case):
    check_case(case)


@pytest.mark.parametrize("case", _DEEP, ids=_ids(_DEEP))
def test_deep_resnet_schedule_matches_reference(case):
    check_case(case)


@pytest.mark.parametrize("case", _BRANCHY_CASES, ids=_ids(_BRANCHY_CASES))
def test_branchy_schedule_matches_reference(case):
    """Configs 3-4: Inception-v4-style branches and DenseNet-121-style k-way
    JOIN-sums (liveness on branches, dense-segment recomputation, peak above
    the floor), full tape parity."""
    check_case(case)


def test_golden_covers_the_hard_paths():
    """The vectors exercise evictions, demand fetches, revives, stalls, fft."""
    seen = set()
    for c in _CASES:
        if "error" in c:
            seen.add("error:" + c["error"][0])
            continue
        r = c["report"]
        if r["evictions"]:
            seen.add("evict")
        if r["demand_transfer_count"]:
            seen.add("demand")
        if r["stall_backup_s"]:
            seen.add("stall_backup")
        if r["stall_prefetch_s"]:
            seen.add("stall_prefetch")
        for e in c.get("tape", ()):
            seen.add("op:" + e[0])
    for need in ["evict", "demand", "stall_backup", "stall_prefetch", "error:SchedulingError",
                 "error:ConfigError", "op:V", "op:P", "op:E", "op:H", "op:X", "op:R"]:
        assert need in seen, need
