"""Benchmark: images/sec of the memory-scheduled training step on B200.

Default workload (BASELINE.json configs[1]): ResNet-50g = gen_resnet(3,4,6,3)
(the reference's generated residual net), batch 256 per GPU, fp32 storage
with tf32 tensor-core math, a 24 GiB pool budget, all five SuperNeurons
features (liveness, offload, LRU cache, cost-aware recompute, conv workspace
selection).  One step = forward + backward + SGD update of one batch.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

Under torchrun each rank is one replica (weak scaling, fixed per-GPU batch)
and the executor sums the weight gradients over NCCL itself, in buckets
overlapped with the backward (dp.py).  Rank 0 prints ONE JSON
line.  ``--impl reference`` times the CPU restatement of the same training
step (oracle/numerics.py; the reference itself has no numerics and cannot
run here) on a bounded sample, with all host threads.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import re
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ALL = "liveness,offload,cache,recompute=cost-aware,convselect"
GiB = 1 << 30


DEFAULT_BATCH = {"resnet50g": 256, "resnet152g": 256, "resnet2534g": 16, "densenet121s": 256, "inception4s": 128,
                 "alexnet": 200, "alex32": 16}
# pool budgets: 24 GiB (BASELINE.json config 2); the depth run uses the
# reference's own 12e9 B at batch 16 (pkg/tests/test_acceptance.py:467-497)
DEFAULT_POOL = {"resnet2534g": 12 * 10 ** 9}
NETS = ["resnet50g", "resnet152g", "resnet2534g", "densenet121s", "inception4s", "alexnet", "alex32"]


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--net", default="resnet50g", choices=NETS,
                    help="benchmark configs: alex32 (1), resnet50g (2, the headline), inception4s (3), "
                         "densenet121s (4), resnet152g / resnet2534g (5)")
    ap.add_argument("--batch", type=int, default=None, help="per-GPU batch (default: the config's)")
    ap.add_argument("--pool-gib", type=float, default=None, help="pool budget in GiB (default: the config's)")
    ap.add_argument("--pool-bytes", type=int, default=None, help="pool budget in bytes (overrides --pool-gib), "
                    "e.g. the schedulable floor max_i(l_i) = 3288334336 for resnet50g b256")
    ap.add_argument("--features", default=ALL)
    ap.add_argument("--stash", default="host", choices=["host", "device"],
                    help="UTP copy-out store: pinned host memory (PCIe) or device HBM (peer / loopback)")
    ap.add_argument("--autotune", action="store_true",
                    help="benchmark the CONV kernel variants per layer shape at create time and run the fastest "
                         "(measured catalog, non-parity mode)")
    ap.add_argument("--precision", default="tf32", choices=["tf32", "fp32"],
                    help="CONV/FC math: tf32 tensor cores (headline) or the fp32-faithful 3xTF32 mode")
    ap.add_argument("--no-extras", action="store_true", help="skip the unconstrained / profile / baseline legs")
    args = ap.parse_args()
    if args.batch is None:
        args.batch = DEFAULT_BATCH[args.net]
    if args.pool_bytes is not None:
        args.pool_gib = args.pool_bytes / GiB
    if args.pool_gib is None:
        args.pool_gib = DEFAULT_POOL.get(args.net, 24 * GiB) / GiB
    return args


def build_net(name: str):
    import paper_1801_04380_b200 as sn
    from paper_1801_04380_b200.netgen import gen_resnet
    if name == "resnet50g":
        return gen_resnet(3, 4, 6, 3)
    if name == "resnet152g":
        return gen_resnet(3, 8, 36, 3)
    if name == "resnet2534g":
        return gen_resnet(211, 211, 211, 211)
    if name == "densenet121s":
        from paper_1801_04380_b200.netgen import gen_densenet
        return gen_densenet()
    if name == "inception4s":
        from paper_1801_04380_b200.netgen import gen_inception
        return gen_inception()
    return sn.load_network(os.path.join(ROOT, "paper_1801_04380_b200", "fixtures", f"{name}.net"))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int) -> None:
        self.index = index
        self.samples: list[list[str]] = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self) -> None:
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def baseline_metric() -> str:
    """BASELINE.json's metric string (the workload itself is in config.workload)."""
    try:
        with open(os.path.join(ROOT, "BASELINE.json")) as fh:
            return json.load(fh)["metric"]
    except (OSError, KeyError, ValueError):
        return "images/sec under memory budget at 1/2/4/8 B200; peak mem vs max_i(l_i)"


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


def tf32_gemm_peaks(device, sustain_s: float = 3.0) -> dict:
    """cuBLAS tf32 GEMM 8192^3 on this box, now: burst (best of 10, CUDA events)
    and sustained (back to back for ``sustain_s`` s, under the power cap) --
    the measured tf32 tensor roofline (MEASURED_PEAKS.json has bf16 only)."""
    import torch
    torch.backends.cuda.matmul.allow_tf32 = True
    n = 8192
    a = torch.randn(n, n, device=device)
    b = torch.randn(n, n, device=device)
    for _ in range(3):
        a @ b
    best = math.inf
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        a @ b
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps, t0 = 0, time.perf_counter()
    s.record()
    while time.perf_counter() - t0 < sustain_s:
        for _ in range(10):
            a @ b
        reps += 10
        torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    sustained = 2 * n ** 3 * reps / (s.elapsed_time(e) / 1e3) / 1e12
    del a, b
    torch.cuda.empty_cache()
    return {"burst": 2 * n ** 3 / (best / 1e3) / 1e12, "sustained": sustained}


def step_traffic(net_name: str, batch: int) -> tuple[dict | None, str]:
    """The per-step DRAM traffic file (tools/launch_table.py merge) for this
    config whose libsnexec digest equals the library this run loads; stale
    files are refused."""
    import glob
    lib_sha = os.path.join(ROOT, "paper_1801_04380_b200", "_lib", "libsnexec.so.sha")
    try:
        digest = open(lib_sha).read().strip()
    except OSError:
        return None, "no libsnexec digest"
    seen = []
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_step_traffic.json"))):
        try:
            d = json.load(open(path))
        except (OSError, ValueError):
            continue
        if d.get("net") != net_name or d.get("batch") != batch or d.get("precision", "tf32") != "tf32":
            continue
        seen.append(os.path.basename(path))
        if d.get("exec_digest") == digest:
            return dict(d, source=os.path.relpath(path, ROOT)), "ok"
    return None, (f"refused {', '.join(seen)}: libsnexec digest differs from this build" if seen
                  else "no traffic capture for this config")


def conv_flops(net, batch: int):
    """Algorithmic tensor FLOPs per iteration: CONV fwd + wgrad + dgrad (dgrad
    skipped when the input is DATA), FC fwd + wgrad + dgrad."""
    import paper_1801_04380_b200 as sn
    shapes = sn.propagate_shapes(net)
    per_layer = {}
    for lay in net.layers:
        if lay.kind not in (sn.LayerKind.CONV, sn.LayerKind.FC):
            continue
        cin_shape = shapes[lay.prev[0]]
        out = shapes[lay.id]
        if lay.kind is sn.LayerKind.CONV:
            k = lay.params["k"]
            mac = batch * out[0] * out[1] * out[2] * cin_shape[0] * k * k
        else:
            mac = batch * out[0] * math.prod(cin_shape)
        has_dgrad = net.layers[lay.prev[0]].kind is not sn.LayerKind.DATA
        per_layer[lay.id] = (2 * mac, 2 * mac * (2 if has_dgrad else 1))  # (fwd, bwd)
    return per_layer


def run_ours(args) -> None:
    import torch
    import paper_1801_04380_b200 as sn
    from paper_1801_04380_b200.training import Executor

    from paper_1801_04380_b200 import dp as dpmod
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    ctx = dpmod.init("nccl")  # torch.distributed: rendezvous, barriers, max-over-ranks timing only
    if world > 1:
        import torch.distributed as dist

    net = build_net(args.net)
    B = args.batch
    pool = args.pool_bytes or int(args.pool_gib * GiB)
    cfg = sn.SimConfig(pool_bytes=pool, features=sn.parse_features(args.features), cost=sn.CostConfig(batch=B))
    free0 = torch.cuda.mem_get_info(local)[0]
    # weight-gradient all-reduce: NCCL buckets inside the executor's step (dp=ctx)
    ex = Executor(net, cfg, device=local, seed=2, lr=0.01, precision=args.precision, dp=ctx if world > 1 else None,
                  stash=args.stash, autotune=args.autotune)
    free1 = torch.cuda.mem_get_info(local)[0]
    rep = ex.report
    c, h, w = sn.propagate_shapes(net)[net.data_id]
    n_cls = math.prod(sn.propagate_shapes(net)[net.terminal_id])
    gen = torch.Generator().manual_seed(1000 + rank)
    images = torch.randn(B, c, h, w, generator=gen)
    labels = torch.randint(0, n_cls, (B,), generator=gen)
    ex.set_inputs(images, labels)
    grads = ex.grads_tensor()

    def step():
        return ex.step(update=True)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kernels = 0
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        start.record()
        losses = []
        for _ in range(args.steps):
            loss, t = step()
            kernels += t.kernels
            losses.append(loss)
        end.record()
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    elapsed_ms = start.elapsed_time(end)
    if dist:
        tt = torch.tensor([elapsed_ms], device=f"cuda:{local}")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed_ms = tt.item()
    ms_per_step = elapsed_ms / args.steps
    value = world * B * args.steps / (elapsed_ms / 1e3)

    # ---- end to end through the public API: pinned host batches in, loss out ----
    # Two pinned host batches used alternately, as a loader's ring would be.
    # Headline: one Executor.step_host_pipelined call per step (batch i+1
    # copied host->device straight into the input buffer while step i computes,
    # the data layer's prefetch; the loss read back at the end of each step);
    # also Executor.train_host over the K steps in one native call
    # (sn_exec_train_host: the loss read back while the next step runs) and the
    # synchronous step_host.  Under the power cap the back-to-back native loop
    # runs at lower SM clocks than the per-step calls, so it is not faster.
    img_host = images.permute(0, 2, 3, 1).contiguous().pin_memory()
    lab_host = labels.to(torch.int32).pin_memory()
    img_host2 = img_host.flip(0).contiguous().pin_memory()
    lab_host2 = lab_host.flip(0).contiguous().pin_memory()
    e_steps = max(3, args.steps)
    ring = [(img_host, lab_host), (img_host2, lab_host2)]
    loop_batches = [ring[i % 2] for i in range(e_steps)]

    def host_step(i, pipelined):
        cur, nxt = ring[i % 2], ring[(i + 1) % 2] if i + 1 < e_steps else (None, None)
        if not pipelined:
            call = lambda upd: ex.step_host(cur[0], cur[1], update=upd)  # noqa: E731
        else:
            call = lambda upd: ex.step_host_pipelined(cur[0], cur[1], nxt[0], nxt[1], update=upd)  # noqa: E731
        return call(True)

    def host_run(pipelined):
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if pipelined == "loop":
            ts = [t.step_ms for _, t in ex.train_host(loop_batches)]
        else:
            ts = [host_step(i, pipelined)[1].step_ms for i in range(e_steps)]
        wall = time.perf_counter() - t0
        if dist:
            tt = torch.tensor([wall], device=f"cuda:{local}")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            wall = tt.item()
        return wall, sum(ts) / len(ts)

    # measured device memory (after the timed region; one extra untimed step)
    mem = ex.memory()
    arena = ex.measure_arena()
    for i in range(2):
        host_step(i, False)
        host_step(i, True)
    # the headline e2e first (right after the device-timed region, before the
    # other host-API variants heat the board further), clocks sampled during it
    with ClockSampler(local) as e2e_clocks:
        e2e_wall, e2e_dev_ms = host_run(True)
    serial_wall, serial_ms = host_run(False)
    ex.train_host(loop_batches[:3])  # untimed warm-up of the native loop
    loop_wall, _ = host_run("loop")
    h2d = img_host.numel() * 4 + lab_host.numel() * 4
    line = {
        "metric": baseline_metric(),
        "value": round(value, 2), "unit": "images/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": ("fp32 storage, tf32 tensor-core math (fp32 accumulate)" if args.precision == "tf32"
                  else "fp32 (3xTF32 split operands on tensor cores, fp32-level products, fp32 accumulate)"),
        "data": "synthetic N(0,1) images, uniform labels; He-uniform weights (seed 2)",
        "config": {"workload": f"{args.net}_b{B}_pool{args.pool_gib:g}GiB_{args.features.replace(',', '+')}"
                               + ("" if args.stash == "host" else "_stash-device"),
                   "model": args.net, "global_batch": B * world, "stash": args.stash, "per_gpu_batch": B, "image": [c, h, w],
                   "parallelism": f"dp{world}", "pool_bytes": pool, "features": args.features,
                   "l2": "no flush needed: per-step working set (~3.3 GB arena) >> 126 MB L2"},
        "e2e": {"value": round(B * world * e_steps / e2e_wall, 2), "unit": "images/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 4,
                "timing": f"host wall clock over {e_steps} Executor.step_host_pipelined calls (max over ranks): "
                          "each step copies its pinned batch host->device (overlapped with the previous step, "
                          "the first one exposed) and reads its loss back",
                "device_images_per_s": round(B * world / (e2e_dev_ms / 1e3), 2), "clocks": e2e_clocks.summary(),
                "train_host_loop_images_per_s": round(B * world * e_steps / loop_wall, 2),
                "serial_step_host_images_per_s": round(B * world / (serial_ms / 1e3), 2),
                "serial_wall_images_per_s": round(B * world * e_steps / serial_wall, 2)},
        "gpu_launches": int(kernels),
        "transfers": dict(ex.transfer_stats(),
                          note="last iteration: offload copy-outs / fetches the tape issued (elided backups "
                               "excluded), copy-engine GB/s, compute-stream time blocked on fetches"),
        "memory": {"peak_bytes": rep.peak_bytes, "min_pool_bytes_max_i_l_i": rep.min_pool_bytes,
                   "peak_over_floor": round(rep.peak_bytes / rep.min_pool_bytes, 4),
                   "pool_high_water_bytes_planned": rep.pool_high_water_bytes,
                   "arena_bytes": mem["arena_bytes"],
                   "arena_written_bytes_measured": arena["measured_arena_written_bytes"],
                   "cudaMemGetInfo_bytes_taken_by_executor": free0 - free1,
                   "device_bytes_over_floor": round((free0 - free1) / rep.min_pool_bytes, 4),
                   "executor_allocations": mem,
                   "baseline_peak_bytes_features_none": rep.baseline_peak_bytes,
                   "offload_d2h_bytes_per_step_issued": int(t.d2h_bytes),
                   "offload_scheduled_bytes_per_step_planned": rep.scheduled_transfer_bytes,
                   "replays_per_step": rep.extra_forward_steps,
                   "conv_wgrad_partials_in_planned_workspace": "%d of %d" % (
                       ex.workspace_use()[0], sum(ex.workspace_use()))},
        "clocks": clocks.summary(),
        **({"autotune_catalog": {"entries": len(ex.catalog()),
                                 "changed_from_default": [f"{c['layer']}:{c['op']}:{c['variant']}" for c in ex.catalog()
                                                          if c["chosen"] and c["variant"] != ex.catalog()[0]["variant"]]}}
           if args.autotune else {}),
        "losses": [round(l, 5) for l in losses[:3]] + [round(losses[-1], 5)],
    }
    # the extras time eager iterations of this executor, whose weight-gradient
    # all-reduce needs every rank: single-replica runs only (the contract asks
    # for roofline / CPU baseline at N = 1)
    if not args.no_extras and world == 1:
        line.update(extras(args, net, cfg, ex, ms_per_step, local))
    ex.close()
    ctx.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def extras(args, net, cfg, ex, ms_per_step, local) -> dict:
    """Roofline of the dominant kernel classes, memory, unconstrained / parity /
    fp32-mode runs, CPU baseline."""
    import torch
    import paper_1801_04380_b200 as sn
    from paper_1801_04380_b200.training import Executor
    out: dict = {}
    # per-action device time of serial eager iterations (weight gradients on
    # the compute stream, so every action's event interval holds exactly its
    # kernels); median of 3
    profs = [ex.profile() for _ in range(3)]
    prof = [(statistics.median(p[i][0] for p in profs), lid, typ) for i, (_, lid, typ) in enumerate(profs[0])]
    flops = conv_flops(net, args.batch)
    t_tensor = f_tensor = t_other = 0.0
    by_kind: dict = {}
    for ms, lid, typ in prof:
        if lid < 0:
            t_other += ms
            continue
        kind = net.layers[lid].kind.value
        key = f"{kind}:{['fwd', 'replay', 'bwd'][typ]}"
        by_kind[key] = by_kind.get(key, 0.0) + ms
        if lid in flops and typ in (0, 2):
            t_tensor += ms
            f_tensor += flops[lid][0 if typ == 0 else 1]
        else:
            t_other += ms
    serial_ms = sum(p[0] for p in prof)
    peaks = measured_peaks()
    # kernel level: every kernel of the iteration replayed node by node with a
    # CUDA event pair around it (median of 5), FLOPs attributed per kernel.
    # Timed BEFORE the cuBLAS peaks: the sustained GEMM leaves the board under
    # its power cap for seconds, and kernels replayed right after it ran ~30 %
    # slower (lower SM clock).  Clocks are sampled during the replay too.
    from paper_1801_04380_b200.profiling import kernel_table
    time.sleep(1.0)
    with ClockSampler(local) as kclocks:
        acts = kernel_table(ex, reps=5)
    tf32 = tf32_gemm_peaks(f"cuda:{local}")
    achieved = f_tensor / (t_tensor / 1e3) / 1e12 if t_tensor else 0.0
    traffic, why = step_traffic(args.net, args.batch)
    tr = traffic["per_step"] if traffic else {}
    ks = [k for a in acts for k in a["kernels"]]
    tk = [k for k in ks if k["flops"] > 0]
    k_us = sum(k["us"] for k in tk)
    k_fl = sum(k["flops"] for k in tk)
    k_ach = k_fl / (k_us / 1e6) / 1e12 if k_us else 0.0
    hk_us = sum(k["us"] for k in ks if k["flops"] == 0)
    top = sorted(ks, key=lambda k: -k["us"])[:8]
    out["roofline"] = {
        "bound": "tensor", "kernel": "CONV/FC implicit-GEMM tcgen05 kind::tf32 kernels (fwd + wgrad + dgrad)",
        "achieved": round(k_ach, 2), "peak": round(tf32["burst"], 2), "unit": "TFLOP/s",
        "frac": round(k_ach / tf32["burst"], 4),
        "peak_source": "cuBLAS tf32 8192^3 burst (best of 10) measured in this run: every kernel is timed alone",
        "how": "achieved = SURVEY 8(d) GEMM FLOPs attributed to the %d tcgen05 kernels of one iteration / their summed "
               "CUDA-event durations (sn_exec_kernel_times: the iteration replayed node by node, an event pair around "
               "each kernel, median of 5, replayed before the cuBLAS peak runs)" % len(tk),
        "kernel_clocks": kclocks.summary(),
        "kernel_us_per_step": round(k_us, 1), "algorithmic_tflop_per_step": round(f_tensor / 1e12, 4),
        "traffic": (tr.get("conv_fc_gemm", {}).get("dram_bytes_per_step") if traffic else None),
        "traffic_source": traffic["source"] if traffic else why,
        "cublas_tf32_sustained": round(tf32["sustained"], 2),
        "bf16_measured_peaks": {k: peaks.get(k) for k in ("bf16_tflops", "bf16_tflops_sustained")},
        "action_level": {"achieved": round(achieved, 2), "frac_of_sustained": round(achieved / tf32["sustained"], 4),
                         "event_ms_per_step": round(t_tensor, 4), "share_of_serial_step": round(t_tensor / serial_ms, 4),
                         "how": "the same FLOPs / the summed event intervals of the CONV/FC tape actions (their "
                                "split-K reductions, weight transposes and bias sums included) in a serial eager "
                                "iteration, against the cuBLAS tf32 sustained peak"},
        "top_kernels": [{"layer": a_name, "kernel": re.sub(r"_GLOBAL__N__[0-9a-f_]+", "", k["name"])[:80],
                         "us": round(k["us"], 1),
                         **({"tflops": round(k["flops"] / (k["us"] / 1e6) / 1e12, 1)} if k["flops"] else {})}
                        for k, a_name in ((k, next(a.get("name", "-") for a in acts if k in a["kernels"])) for k in top)]}
    hbm_peak = float(peaks.get("hbm_gbs") or 6650.0)
    hl = tr.get("hbm_layers") if traffic else None
    out["roofline_hbm_layers"] = {
        "bound": "hbm", "kernel": "BN / ReLU / JOIN / POOL / softmax / split-K / SGD layer kernels",
        "kernel_us_per_step": round(hk_us, 1), "event_ms_per_step_actions": round(t_other, 4), "peak": hbm_peak,
        "unit": "GB/s",
        "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks.get("hbm_gbs") else "B200_PROFILING.md fallback",
        "traffic": hl["dram_bytes_per_step"] if hl else None,
        "traffic_source": traffic["source"] if traffic else why}
    if hl and hk_us:
        gbs = hl["dram_bytes_per_step"] / (hk_us / 1e6) / 1e9
        out["roofline_hbm_layers"].update(achieved=round(gbs, 1), frac=round(gbs / hbm_peak, 4),
                                          how="ncu DRAM bytes of these launches (same libsnexec digest) / their "
                                              "summed CUDA-event durations this run (kernel replay, median of 5)")
    hb = tr.get("hbm_bulk") if traffic else None
    if hb and hb.get("flat_kernel_indices") and len(ks) == traffic.get("launches"):
        b_us = sum(ks[i]["us"] for i in hb["flat_kernel_indices"])
        gbs = hb["dram_bytes_per_step"] / (b_us / 1e6) / 1e9
        out["roofline_hbm_layers"]["bulk"] = {
            "launches": hb["launches"], "min_bytes_per_launch": hb["min_bytes_per_launch"],
            "traffic": hb["dram_bytes_per_step"], "kernel_us_per_step": round(b_us, 1), "achieved": round(gbs, 1),
            "frac": round(gbs / hbm_peak, 4),
            "how": "the HBM launches moving >= 50 MB each (BN statistics / dx passes, BN apply + JOIN, pool, stem "
                   "pad): their ncu DRAM bytes / their summed CUDA-event durations this run; the rest of the class is "
                   "short latency-bound launches (finalisers, tile statistics, weight transposes, split-K reductions)"}
    out["time_by_layer_kind_ms"] = {k: round(v, 3) for k, v in sorted(by_kind.items(), key=lambda kv: -kv[1])}

    def side_run(label, cfg2, steps=5, **kw):
        try:
            sex = Executor(net, cfg2, device=local, seed=2, **kw)
            sex.set_inputs(*_inputs(net, args.batch))
            for _ in range(3):
                sex.step()
            ms = statistics.median(sex.step()[1].step_ms for _ in range(steps))
            extra = {"transfers": sex.transfer_stats()}
            sex.close()
            return ms, extra
        except Exception as exc:  # report, never hide
            return None, {"error": f"{label}: {str(exc)[:200]}"}

    # unconstrained reference run: all features off, pool = whole-iteration
    # residency.  The step runs under the power cap, so its clock depends on
    # what ran just before: both executors are timed the same way, in
    # alternating blocks of back-to-back steps (CUDA events, median block),
    # and the overhead is their ratio -- not the headline loop against a side run.
    base_pool = ex.report.baseline_peak_bytes + (256 << 20)
    out["unconstrained"] = {"features": "none", "pool_bytes": base_pool}
    try:
        uex_ = Executor(net, sn.SimConfig(pool_bytes=base_pool, features=sn.Features(), cost=cfg.cost), device=local,
                        seed=2)
        uex_.set_inputs(*_inputs(net, args.batch))

        def block(e, n=5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            for _ in range(n):
                e.step(update=False)
            b.record()
            torch.cuda.synchronize()
            return a.elapsed_time(b) / n

        for e in (ex, uex_):
            block(e, 3)
        sched, unc = [], []
        for _ in range(4):
            sched.append(block(ex))
            unc.append(block(uex_))
        uex_.close()
        ms_s, ms_u = statistics.median(sched), statistics.median(unc)
        out["unconstrained"].update(
            ms_per_step=round(ms_u, 4), scheduled_ms_per_step_same_method=round(ms_s, 4),
            overhead_of_memory_schedule=round(ms_s / ms_u - 1.0, 4),
            how="4 alternating blocks of 5 back-to-back steps per executor (no update), CUDA events, median block")
    except Exception as exc:  # report, never hide
        out["unconstrained"]["error"] = str(exc)[:200]
    # parity mode: every copy-out the reference schedules is issued
    pm, pex = side_run("parity", cfg, elide_backups=False)
    out["parity_mode"] = {"elide_backups": False, "ms_per_step": pm and round(pm, 4),
                          "images_per_s": pm and round(args.batch / (pm / 1e3), 2), **pex}
    # the Unified Tensor Pool's copy-out store in HBM (f2: an NVLink peer's spare
    # memory; on one GPU the same device as a loopback) vs pinned host memory,
    # at a pool tight enough that the schedule fetches tensors back (4 GiB)
    tight = sn.SimConfig(pool_bytes=4 * GiB, features=cfg.features, cost=cfg.cost)
    th, thx = side_run("host stash", tight)
    td, tdx = side_run("device stash", tight, stash="device")
    out["utp_stash"] = {"pool_bytes": 4 * GiB,
                        "host_pinned": {"ms_per_step": th and round(th, 4),
                                        "images_per_s": th and round(args.batch / (th / 1e3), 2), **thx},
                        "device_loopback": {"ms_per_step": td and round(td, 4),
                                            "images_per_s": td and round(args.batch / (td / 1e3), 2), **tdx},
                        "note": "stash=device on this GPU stands in for a peer's HBM over NVLink (unmeasured at "
                                "N>1: one GPU per run here)"}
    # fp32-faithful numerics (3xTF32 split operands) at the same config
    fm, fex = side_run("fp32", cfg, precision="fp32")
    out["fp32_mode"] = {"precision": "fp32 (3xTF32 split operands, fp32-level products)",
                        "ms_per_step": fm and round(fm, 4),
                        "images_per_s": fm and round(args.batch / (fm / 1e3), 2),
                        **({"error": fex["error"]} if "error" in fex else {})}
    out["cpu_baseline"] = cpu_baseline(args.net, sample=min(args.batch, 16))
    return out


def _inputs(net, B):
    import torch
    from oracle import netdef
    onet = netdef.as_onet(net)
    shp = netdef.shapes(onet)
    c, h, w = shp[onet.data_id]
    n_cls = math.prod(shp[onet.terminal_id])
    g = torch.Generator().manual_seed(1000)
    return torch.randn(B, c, h, w, generator=g), torch.randint(0, n_cls, (B,), generator=g)


def net_text(name: str) -> str:
    """The config's ``.net`` text without the product package: the oracle's
    restated generator for the residual nets, the bundled text files otherwise."""
    from oracle import netdef
    blocks = {"resnet50g": (3, 4, 6, 3), "resnet152g": (3, 8, 36, 3), "resnet2534g": (211, 211, 211, 211)}
    if name in blocks:
        return netdef.resnet_text(*blocks[name])
    with open(os.path.join(ROOT, "paper_1801_04380_b200", "fixtures", f"{name}.net")) as fh:
        return fh.read()


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline(name: str, sample: int) -> dict:
    """The CPU restatement (oracle/numerics.py, no product code) timed on the
    host cores on a bounded sample of the workload."""
    import torch
    from oracle import netdef
    from oracle.numerics import forward_backward
    threads = len(os.sched_getaffinity(0))
    torch.set_num_threads(threads)
    onet = netdef.parse_net(net_text(name), name)
    params = netdef.init_parameters(onet, seed=2)
    images, labels = _inputs(onet, sample)
    forward_backward(onet, params, images, labels)  # warm
    t0 = time.perf_counter()
    reps = 0
    while reps < 2 or time.perf_counter() - t0 < 5.0:
        forward_backward(onet, params, images, labels)
        reps += 1
        if time.perf_counter() - t0 > 25.0:
            break
    dt = (time.perf_counter() - t0) / reps
    return {"value": round(sample / dt, 3), "unit": "images/s", "cores": threads, "kind": "port",
            "cpu": cpu_model(),
            "sample": f"{reps} fp32 fwd+bwd passes of {sample} images ({name}), torch CPU restatement "
                      "(oracle/numerics.py)"}


def run_reference(args) -> None:
    """The reference's CPU path for this workload, on the host cores, with no
    product code: (1) the training step the reference describes but cannot
    execute (it has no tensors), as the oracle's torch CPU fp32
    restatement, full per-GPU batch per step; (2) the unmodified reference
    package's own schedule computation (memsched.run_simulation from
    baseline/_ref) for the same config."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch
    from oracle import netdef
    from oracle.numerics import forward_backward, sgd_step
    threads = len(os.sched_getaffinity(0))
    torch.set_num_threads(threads)
    text = net_text(args.net)
    onet = netdef.parse_net(text, args.net)
    B = args.batch
    params = netdef.init_parameters(onet, seed=2)
    images, labels = _inputs(onet, B)
    for _ in range(max(1, args.warmup)):
        forward_backward(onet, params, images, labels)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        _, grads = forward_backward(onet, params, images, labels)
        params = sgd_step(params, grads, 0.01)
    dt = time.perf_counter() - t0
    value = B * args.steps / dt
    pool = int(args.pool_gib * GiB)
    print(json.dumps({
        "impl": "reference", "metric": baseline_metric(), "value": round(value, 3), "unit": "images/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": max(1, args.warmup),
        "ms_per_step": round(dt / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
        "data": "synthetic N(0,1) images, uniform labels; He-uniform weights (seed 2)",
        "config": {"workload": f"{args.net}_b{B}_pool{args.pool_gib:g}GiB_{args.features.replace(',', '+')}",
                   "model": args.net, "global_batch": B, "per_gpu_batch": B, "parallelism": "cpu",
                   "pool_bytes": pool, "features": args.features},
        "cpu_baseline": {"value": round(value, 3), "unit": "images/s", "cores": threads, "kind": "port",
                         "cpu": cpu_model(),
                         "sample": f"full {args.net} batch of {B} per step, fwd+bwd+SGD, torch CPU fp32 "
                                   "restatement oracle/numerics.py (the reference memsched package is a simulator "
                                   "with no tensor numerics)"},
        "e2e": {"value": round(value, 3), "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_simulator": reference_simulator_time(args, text, pool),
    }), flush=True)


def reference_simulator_time(args, text: str, pool: int) -> dict:
    """The unmodified reference package (memsched 0.1.0, installed offline into
    baseline/_ref with --no-deps: matplotlib is only for its PNG figures)
    planning this config with its own run_simulation -- the reference's CPU
    path for the schedule (1 core, CPython)."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "memsched")):
        return {"unavailable": "baseline/_ref not installed"}
    sys.path.insert(0, ref_dir)
    try:
        import memsched
        rnet = memsched.parse_network(text, name=args.net)
        cfg = memsched.SimConfig(pool_bytes=pool, features=memsched.parse_features(args.features),
                                 cost=memsched.CostConfig(batch=args.batch))
        times = []
        for _ in range(1 if len(rnet.layers) > 1000 else 3):
            t0 = time.perf_counter()
            rep = memsched.run_simulation(rnet, cfg)
            times.append(time.perf_counter() - t0)
        return {"run_simulation_s": round(statistics.median(times), 4), "cores": 1, "cpu": cpu_model(),
                "module": os.path.relpath(memsched.__file__, ROOT),
                "peak_bytes": rep.peak_bytes, "min_pool_bytes": rep.min_pool_bytes,
                "pool_high_water_bytes": rep.pool_high_water_bytes}
    except Exception as exc:  # report, never hide
        return {"error": str(exc)[:200]}
    finally:
        sys.path.remove(ref_dir)


def main() -> None:
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
