"""Generate the schedule-parity golden vectors from the reference simulator.

Run in the build container only (the reference is not present on GPU boxes):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

For every case it records the inputs (network text, batch, pool, features,
cost overrides) and the reference outputs of ``memsched.run_simulation``:
every ``SimReport`` field, the rows, the conv-algorithm selections, and the
physical event tape (block-pool allocs/frees with offsets, copy-outs,
fetches, replays, compute points, LRU cache operations), captured by
subclassing the reference's ``_Simulation`` without modifying it.

Large row/tape payloads are stored as a SHA-256 of their canonical JSON;
small ones are stored in full so a mismatch can be diagnosed on any box.
Output: ``tests/golden/sched_golden.json.gz``.
"""

from __future__ import annotations

import dataclasses
import gzip
import hashlib
import json
import sys
import time
from pathlib import Path

import memsched
from memsched import netgen, simulator as refsim
from memsched.cli import resolve_network
from memsched.costmodel import baseline_peak_bytes, build_costs

HERE = Path(__file__).resolve().parent
OUT = HERE / "sched_golden.json.gz"
ALEX32 = (HERE.parent.parent / "paper_1801_04380_b200" / "fixtures" / "alex32.net").read_text()

MiB = 1 << 20
GiB = 1 << 30
FULL_LIMIT = 4000  # events/rows above this are stored as digests only

FEATURES = [
    "none", "liveness", "liveness,offload", "liveness,offload,recompute=speed",
    "liveness,offload,recompute=memory", "cache,recompute=cost-aware",
    "liveness,offload,cache,recompute=cost-aware,convselect",
]
EXTRA_FEATURES = [
    "liveness,convselect", "offload,cache", "recompute=speed", "recompute=memory",
    "cache,recompute=speed,convselect", "cache,recompute=memory,convselect",
    "offload,convselect", "cache,convselect",
]
ALL = "liveness,offload,cache,recompute=cost-aware,convselect"


class TapeSim(refsim._Simulation):
    """Reference simulation that also records the physical event tape."""

    def __init__(self, net, config):
        super().__init__(net, config)
        self.tape: list[list] = []
        pool, cache, tape = self.pool, self.cache, self.tape
        p_alloc, p_free = pool.alloc, pool.free

        def alloc(key, nbytes, high=False):
            off = p_alloc(key, nbytes, high=high)
            tape.append(["A", key[0], key[1], off, pool._allocated[key][1], int(high)])
            return off

        def free(key):
            p_free(key)
            tape.append(["F", key[0], key[1]])

        pool.alloc, pool.free = alloc, free
        c_insert, c_discard, c_evict = cache.insert, cache.discard, cache.evict_lru

        def insert(key, nbytes):
            tape.append(["T" if key in cache else "I", key[1]])
            c_insert(key, nbytes)

        def discard(key):
            if key in cache:
                tape.append(["X", key[1]])
            return c_discard(key)

        def evict_lru():
            key, nbytes = c_evict()
            tape.append(["E", key[1]])
            return key, nbytes

        cache.insert, cache.discard, cache.evict_lru = insert, discard, evict_lru

    def _copy_out(self, lid):
        self.tape.append(["O", lid])
        super()._copy_out(lid)

    def _fetch_scheduled(self, lid):
        self.tape.append(["P", lid])
        super()._fetch_scheduled(lid)

    def _fetch_demand(self, lid):
        self.tape.append(["D", lid])
        super()._fetch_demand(lid)

    def _materialize(self, lid, nbytes):
        key = ("act", lid)
        hit = key in self.cache
        revive = (not hit) and key in self.pool
        out = super()._materialize(lid, nbytes)
        if hit:
            self.tape.append(["H", lid])
        elif revive:
            self.tape.append(["V", lid])
        return out

    def _replay_member(self, mid, replay_rows):
        before = self.extra_steps
        super()._replay_member(mid, replay_rows)
        if self.extra_steps != before:
            self.tape.append(["R", mid])

    def _select_workspace(self, s, layer, cost, phase):
        n_sel = len(self.selections)
        mult, ws_key = super()._select_workspace(s, layer, cost, phase)
        algo = self.selections[-1].algo if len(self.selections) > n_sel else ""
        self.tape.append(["C" if phase == "forward" else "B", layer.id, algo,
                          -1 if ws_key is None else ws_key[1]])
        return mult, ws_key

    def _end_of_step(self, s):
        super()._end_of_step(s)
        self.tape.append(["S", s])


def canon(obj) -> str:
    return json.dumps(obj, separators=(",", ":"), sort_keys=False)


def digest(obj) -> str:
    return hashlib.sha256(canon(obj).encode()).hexdigest()


def report_dict(rep) -> dict:
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


def capture_text(fn, *args, **kw):
    """Run a reference generator and capture the text it parsed."""
    seen = {}
    orig = netgen.parse_network

    def spy(text, name="net"):
        seen["text"], seen["name"] = text, name
        return orig(text, name=name)

    netgen.parse_network = spy
    try:
        fn(*args, **kw)
    finally:
        netgen.parse_network = orig
    return seen["text"], seen["name"]


def fixture_text(name: str) -> str:
    from importlib import resources
    return (resources.files("memsched") / "fixtures" / f"{name}.net").read_text()


def run_case(case: dict) -> dict:
    net = memsched.parse_network(case["text"], name=case["name"])
    cost = memsched.CostConfig(batch=case["batch"], **case.get("cost", {}))
    out = dict(case)
    try:
        cfg = memsched.SimConfig(pool_bytes=case["pool"],
                                 features=memsched.parse_features(case["features"]),
                                 cost=cost)
        sim = TapeSim(net, cfg)
        rep = sim.run()
    except memsched.MemschedError as exc:
        out["error"] = [type(exc).__name__, str(exc)]
        return out
    rd = report_dict(rep)
    rows, sels = rd.pop("rows"), rd.pop("selections")
    out["report"] = rd
    out["rows_sha"] = digest(rows)
    out["sel_sha"] = digest(sels)
    out["tape_sha"] = digest(sim.tape)
    out["tape_len"] = len(sim.tape)
    if len(rows) <= FULL_LIMIT:
        out["rows"] = rows
        out["selections"] = sels
    if len(sim.tape) <= FULL_LIMIT:
        out["tape"] = sim.tape
    return out


def cases() -> list[dict]:
    out: list[dict] = []
    alex = fixture_text("alexnet")

    def add(cid, text, name, batch, pool, feats, **cost):
        c = {"id": cid, "text": text, "name": name, "batch": batch, "pool": pool,
             "features": feats}
        if cost:
            c["cost"] = cost
        out.append(c)

    # AlexNet fixture, the reference's own calibration matrix and beyond.
    for f in FEATURES + EXTRA_FEATURES:
        add(f"alexnet/b200/4GiB/{f}", alex, "alexnet", 200, 4 * GiB, f)
    for mib_ in [1250, 1350, 1500, 1750, 2048, 2560, 3072, 4096, 6144]:
        add(f"alexnet/all/{mib_}MiB", alex, "alexnet", 200, mib_ * MiB, ALL)
    for b in [50, 100, 150, 200, 210, 230, 250]:
        add(f"alexnet/knee/b{b}", alex, "alexnet", b, 1536 * MiB, "cache")
    for b in [50, 100, 150, 200]:
        add(f"alexnet/offload/b{b}", alex, "alexnet", b, 4 * GiB, "liveness,offload")
    add("alexnet/err/floor", alex, "alexnet", 200, 600 * MiB, "offload,recompute=memory")
    add("alexnet/err/100MiB", alex, "alexnet", 200, 100 * MiB, "none")
    add("alexnet/err/oom", alex, "alexnet", 200, GiB, "none")
    # Slow / fast links exercise pending backed drops, backup and demand stalls.
    for bw in [5e7, 5e8, 2e9, 3.3e10]:
        for f in FEATURES[2:] + EXTRA_FEATURES[1:]:
            add(f"alexnet/bw{bw:g}/{f}", alex, "alexnet", 200, 4 * GiB, f,
                bandwidth_bytes_per_s=bw)
    for pool_mib in range(890, 1600, 37):
        for f in ["cache,recompute=cost-aware", ALL, "cache,recompute=speed,convselect",
                  "cache,recompute=memory", "offload,cache,convselect"]:
            add(f"alexnet/tight/{pool_mib}/{f}", alex, "alexnet", 200, pool_mib * MiB, f,
                bandwidth_bytes_per_s=1e9)

    # alex32 (config 1).
    for f in FEATURES + EXTRA_FEATURES:
        add(f"alex32/b16/1GiB/{f}", ALEX32, "alex32", 16, GiB, f)
    for pool in [16777216, 17 * MiB, 20 * MiB, 24 * MiB, 28 * MiB]:
        for f in [ALL, "cache,recompute=memory", "cache,recompute=speed,convselect"]:
            add(f"alex32/tight/{pool}/{f}", ALEX32, "alex32", 16, pool, f)
            add(f"alex32/tight/{pool}/slow/{f}", ALEX32, "alex32", 16, pool, f,
                bandwidth_bytes_per_s=1e8)

    # Branching fixtures.
    for fx in ["fan12", "nested_fan10"]:
        text = fixture_text(fx)
        for b in [8, 32]:
            net = memsched.parse_network(text, name=fx)
            base = baseline_peak_bytes(build_costs(net, memsched.CostConfig(batch=b)))
            for f in FEATURES + EXTRA_FEATURES:
                add(f"{fx}/b{b}/roomy/{f}", text, fx, b, 2 * base + 64 * MiB, f)
                add(f"{fx}/b{b}/tight/{f}", text, fx, b, base // 2, f,
                    bandwidth_bytes_per_s=1e8)

    # Uniform chains (closed forms of the reference's criterion 1).
    chain_tensor = 4 * 16 * 16 * 4 * 200
    for n, cps in [(9, (3, 6)), (12, (3, 6, 9)), (7, ()), (10, (1, 10))]:
        text, name = capture_text(netgen.make_uniform_chain, n, cps)
        for f in FEATURES:
            add(f"chain{n}{cps}/{f}", text, name, 200, 4 * n * chain_tensor, f)

    # Random fan-join nets.
    for seed in range(200):
        text, name = capture_text(netgen.random_fanjoin, seed)
        net = memsched.parse_network(text, name=name)
        base = baseline_peak_bytes(build_costs(net, memsched.CostConfig(batch=8)))
        for f in ["none", "liveness", "liveness,offload", "liveness,offload,recompute=memory",
                  ALL]:
            add(f"fanjoin{seed}/{f}", text, name, 8, 2 * base + 64 * MiB, f)
        if seed < 60:
            for f in [ALL, "cache,recompute=speed", "cache,recompute=memory,convselect"]:
                for frac in (3, 5):
                    add(f"fanjoin{seed}/tight{frac}/{f}", text, name, 8, base * 2 // frac, f,
                        bandwidth_bytes_per_s=2e7)

    # Generated residual networks (configs 2 and 5).
    r50, r50n = capture_text(netgen.gen_resnet, 3, 4, 6, 3)
    for f in FEATURES + ["cache,recompute=speed,convselect", "cache,recompute=memory,convselect"]:
        add(f"resnet50g/b256/24GiB/{f}", r50, r50n, 256, 24 * GiB, f)
    for pool in [3288334336, 3500 * MiB, 4 * GiB, 5 * GiB]:
        add(f"resnet50g/b256/tight{pool}/all", r50, r50n, 256, pool, ALL)
        add(f"resnet50g/b256/tight{pool}/all/slow", r50, r50n, 256, pool, ALL,
            bandwidth_bytes_per_s=1e9)
    add("resnet50g/b32/all", r50, r50n, 32, 24 * GiB, ALL)
    r152, r152n = capture_text(netgen.gen_resnet, 3, 8, 36, 3)
    for f in ["none", ALL, "liveness,offload,recompute=memory"]:
        add(f"resnet152g/b256/180GiB/{f}", r152, r152n, 256, 180 * GiB, f)
    r830, r830n = capture_text(netgen.gen_resnet, 69, 69, 69, 69)
    add("resnet830g/b16/none", r830, r830n, 16, 12 * 10 ** 9, "none")
    r842, r842n = capture_text(netgen.gen_resnet, 70, 70, 70, 70)
    add("resnet842g/b16/none", r842, r842n, 16, 12 * 10 ** 9, "none")
    r2534, r2534n = capture_text(netgen.gen_resnet, 211, 211, 211, 211)
    add("resnet2534g/b16/all", r2534, r2534n, 16, 12 * 10 ** 9, ALL)
    return out


def analysis_case(text: str, name: str, batch: int) -> dict:
    """Every analysis entry point of the reference API on one network."""
    from memsched import liveness as lv, offload as ol, recompute as rc
    net = memsched.parse_network(text, name=name)
    costs = build_costs(net, memsched.CostConfig(batch=batch))
    sched = memsched.build_schedule(net)
    out: dict = {"text": text, "name": name, "batch": batch}
    out["forward_ids"] = sched.forward_ids
    out["costs"] = [[list(c.shape), c.out_elems, c.out_bytes, c.device_bytes, c.grad_bytes, c.param_bytes,
                     c.fwd_time, c.bwd_time] for c in costs.values()]
    out["fwd_uses"] = {str(k): v for k, v in lv.forward_use_steps(net, sched).items()}
    out["bwd_uses"] = {str(k): v for k, v in lv.backward_use_steps(net, sched).items()}
    out["last_use"] = {str(k): v for k, v in lv.last_use_step(net, sched).items()}
    out["last_fwd_use"] = {str(k): v for k, v in lv.last_forward_use_step(net, sched).items()}
    for seed in (False, True):
        out[f"grad_buffers_{int(seed)}"] = [dataclasses.astuple(b) for b in
                                             lv.grad_buffers(net, costs, sched, seed).values()]
    out["liveness_table"] = [dataclasses.astuple(r) for r in lv.liveness_table(net, costs, sched)]
    out["liveness_csv"] = lv.dump_liveness_csv(net, costs, sched)
    out["curve_liveness"] = lv.resident_curve(net, costs, sched, "liveness")
    out["curve_baseline"] = lv.resident_curve(net, costs, sched, "baseline")
    out["liveness_peak"] = list(lv.liveness_peak(net, costs, sched))
    bufs = lv.grad_buffers(net, costs, sched, False)
    out["working_set"] = [lv.working_set_bytes(net, costs, sched, bufs, s) for s in range(sched.num_steps)]
    op = ol.build_offload_plan(net, sched)
    out["offload_plan"] = [list(op.cp_ids), {str(k): v for k, v in op.drop_after.items()},
                           {str(k): v for k, v in op.prefetch_issue.items()},
                           {str(k): v for k, v in op.first_backward_use.items()},
                           {str(k): v for k, v in op.last_backward_use.items()}]
    segs = rc.build_segments(net, sched)
    out["segments"] = [[s.index, list(s.members), list(s.anchors), rc.first_backward_use(net, sched, s),
                        rc.memory_extras(net, s), rc.speed_extras(net, sched, s),
                        rc.speed_prediction(net, costs, sched, s)] for s in segs]
    plans = {}
    for pol in rc.POLICIES:
        for off in (False, True):
            p = rc.plan(net, costs, sched, pol, frozenset(op.cp_ids) if off else frozenset())
            plans[f"{pol}/{int(off)}"] = [list(p.modes), sorted(p.spill_ids), p.extra_forward_steps,
                                         list(p.predictions)]
    out["plans"] = plans
    out["step_demands"] = rc.step_demands(net, costs, sched)
    dp = rc.demand_peak(net, costs, sched)
    out["demand_peak"] = [dp.nbytes, dp.step, dp.layer_id]
    return out


def pool_trace(seed: int, ops: int, capacity_blocks: int) -> dict:
    """A random alloc/free trace through the reference BlockPool."""
    import random
    from memsched.poolalloc import BLOCK_BYTES, BlockPool, PoolExhausted
    pool = BlockPool(capacity_blocks * BLOCK_BYTES)
    rng = random.Random(seed)
    live, trace, nxt = [], [], 0
    for _ in range(ops):
        if live and rng.random() < 0.4:
            key = live.pop(rng.randrange(len(live)))
            pool.free(key)
            trace.append(["F", key])
        else:
            key, nxt = nxt, nxt + 1
            nbytes = rng.randrange(0, 40 * BLOCK_BYTES)
            high = rng.random() < 0.3
            try:
                off = pool.alloc(key, nbytes, high=high)
                live.append(key)
            except PoolExhausted as exc:
                off = str(exc)
            trace.append(["A", key, nbytes, int(high), off, pool.used_bytes, pool.high_water_bytes])
    return {"seed": seed, "capacity_blocks": capacity_blocks, "trace": trace}


def main() -> None:
    t0 = time.time()
    results = []
    texts: dict[str, str] = {}
    for case in cases():
        res = run_case(case)
        # De-duplicate network texts to keep the file small.
        key = hashlib.sha256(res["text"].encode()).hexdigest()[:16]
        texts[key] = res.pop("text")
        res["net"] = key
        results.append(res)
    payload = {"generator": "tests/golden/make_golden.py",
               "reference": "memsched 0.1.0 (/root/reference/pkg)",
               "python": sys.version.split()[0],
               "nets": texts, "cases": results}
    with gzip.open(OUT, "wt") as fh:
        json.dump(payload, fh, separators=(",", ":"))
    # analysis entry points + allocator traces
    nets = [(fixture_text("alexnet"), "alexnet", 200), (ALEX32, "alex32", 16),
            (fixture_text("fan12"), "fan12", 8), (fixture_text("nested_fan10"), "nested_fan10", 4)]
    nets.append(capture_text(netgen.gen_resnet, 3, 4, 6, 3) + (256,))
    for n, cps in [(9, (3, 6)), (12, (3, 6, 9))]:
        nets.append(capture_text(netgen.make_uniform_chain, n, cps) + (200,))
    for seed in range(0, 200, 10):
        nets.append(capture_text(netgen.random_fanjoin, seed) + (8,))
    analysis = [analysis_case(t, n, b) for t, n, b in nets]
    traces = [pool_trace(90210, 20000, 256), pool_trace(577, 2000, 64), pool_trace(1, 5000, 1024)]
    with gzip.open(HERE / "analysis_golden.json.gz", "wt") as fh:
        json.dump({"generator": "tests/golden/make_golden.py", "analysis": analysis, "pool_traces": traces}, fh,
                  separators=(",", ":"))
    n_err = sum(1 for r in results if "error" in r)
    print(f"{len(results)} cases ({n_err} errors) in {time.time() - t0:.1f}s -> {OUT}")


BRANCHY_OUT = HERE / "sched_golden_branchy.json.gz"


def branchy_cases() -> list[dict]:
    """Benchmark configs 3 and 4: the Inception-v4-style (branches, 4-way
    JOIN-sum) and DenseNet-121-style (k-way JOIN-sum, dense recomputation)
    graphs of paper_1801_04380_b200/netgen.py -- the reference ships no
    generator for them, so their text is produced by ours and scheduled by the
    reference."""
    sys.path.insert(0, str(HERE.parent.parent))
    from paper_1801_04380_b200 import netgen as ours
    out: list[dict] = []
    nets = [("densenet121s", ours.densenet_text(), 256), ("inception4s", ours.inception_text(), 128),
            ("densenet_small", ours.densenet_text(blocks=(2, 3, 2, 2), widths=(32, 64, 64, 64)), 8),
            ("inception_small", ours.inception_text(n_a=1, n_b=1, n_c=1), 4)]
    for name, text, b in nets:
        net = memsched.parse_network(text, name=name)
        base = baseline_peak_bytes(build_costs(net, memsched.CostConfig(batch=b)))
        for f in FEATURES + ["cache,recompute=speed,convselect", "cache,recompute=memory,convselect"]:
            out.append({"id": f"{name}/b{b}/roomy/{f}", "text": text, "name": name, "batch": b,
                        "pool": base + 256 * MiB, "features": f})
        for frac in (2, 3):
            for f in [ALL, "cache,recompute=memory,convselect"]:
                out.append({"id": f"{name}/b{b}/tight{frac}/{f}", "text": text, "name": name, "batch": b,
                            "pool": base // frac, "features": f, "cost": {"bandwidth_bytes_per_s": 2e9}})
    return out


def main_branchy() -> None:
    t0 = time.time()
    results, texts = [], {}
    for case in branchy_cases():
        res = run_case(case)
        key = hashlib.sha256(res["text"].encode()).hexdigest()[:16]
        texts[key] = res.pop("text")
        res["net"] = key
        results.append(res)
    with gzip.open(BRANCHY_OUT, "wt") as fh:
        json.dump({"generator": "tests/golden/make_golden.py --branchy",
                   "reference": "memsched 0.1.0 (/root/reference/pkg)", "python": sys.version.split()[0],
                   "nets": texts, "cases": results}, fh, separators=(",", ":"))
    n_err = sum(1 for r in results if "error" in r)
    print(f"{len(results)} cases ({n_err} errors) in {time.time() - t0:.1f}s -> {BRANCHY_OUT}")


if __name__ == "__main__":
    if "--branchy" in sys.argv:
        main_branchy()
    else:
        main()
