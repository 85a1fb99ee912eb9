"""Unit checks of planner internals that the golden vectors exercise only
indirectly: the CPython set-order emulation, the C-ABI surface, timing.
"""

from __future__ import annotations

import ctypes as C
import random
import re
import time
from pathlib import Path

import pytest

import paper_1801_04380_b200 as sn
from paper_1801_04380_b200 import _cabi, _native

ROOT = Path(__file__).resolve().parents[1]


def _pyset_native(a, b, a2):
    L = _cabi.lib()
    arr = lambda v: (C.c_int64 * max(1, len(v)))(*v)
    n = C.c_size_t()
    out = (C.c_int64 * 4096)()
    rc = L.sn_debug_pyset(arr(a), len(a), arr(b), len(b), arr(a2), len(a2), out, 4096, C.byref(n))
    assert rc == 0
    return list(out[: n.value])


@pytest.mark.parametrize("seed", range(300))
def test_pyset_iteration_order_matches_cpython(seed):
    rng = random.Random(seed)
    hi = rng.choice([8, 16, 40, 200, 5000])
    a = [rng.randrange(hi) for _ in range(rng.randrange(0, 30))]
    b = [rng.randrange(hi) for _ in range(rng.randrange(0, 30))]
    a2 = [rng.randrange(hi) for _ in range(rng.randrange(0, 10))]
    s, t = set(), set()
    for x in a:
        s.add(x)
    for x in b:
        t.add(x)
    s.update(t)
    for x in a2:
        s.add(x)
    assert _pyset_native(a, b, a2) == list(s)


def _header_symbols():
    text = (ROOT / "include" / "superneurons.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sn_[a-z0-9_]+)\s*\(", text)))


def test_c_abi_exports_every_declared_symbol():
    """Both libraries load without a GPU and export what the header declares."""
    plan = _native.planner()
    exe = _native.executor()
    missing = []
    for sym in _header_symbols():
        lib = exe if sym.startswith(("sn_exec", "sn_dp")) else plan
        if not hasattr(lib, sym):
            missing.append(sym)
    assert not missing, missing


def test_planner_is_fast_on_the_deepest_config():
    """ResNet-2534g b16: the reference takes ~6.4 s; the planner ms."""
    from paper_1801_04380_b200.netgen import gen_resnet
    net = gen_resnet(211, 211, 211, 211)
    cfg = sn.SimConfig(pool_bytes=12 * 10 ** 9,
                       features=sn.parse_features("liveness,offload,cache,recompute,convselect"),
                       cost=sn.CostConfig(batch=16))
    t0 = time.perf_counter()
    rep = sn.run_simulation(net, cfg)
    elapsed = time.perf_counter() - t0
    assert rep.peak_bytes == 205520896
    assert elapsed < 2.0
