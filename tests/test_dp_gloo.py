"""World-size-2 data parallelism on CPU (gloo): the DP plumbing used by
bench.py on NCCL, checked with the CPU oracle standing in for the executor.

Two replicas on disjoint halves of a batch, gradients summed by
``dp.average_gradients`` and scaled by 1/world, must equal the gradient of
the full-batch mean loss (alex32 has no BatchNorm, so per-replica batch
statistics do not enter; dropout runs at rate 0 because its hash mask is a
function of the element index inside each replica's batch).  Every rank must
also plan the identical schedule.
"""

from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _net(sn):
    path = os.path.join(ROOT, "paper_1801_04380_b200", "fixtures", "alex32.net")
    text = open(path).read().replace(" DROPOUT", " DROPOUT rate=0.0")
    return sn.parse_network(text, name="alex32")


def _worker(rank: int, world: int, port: int, out_q) -> None:
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    torch.set_num_threads(1)
    import paper_1801_04380_b200 as sn
    from paper_1801_04380_b200 import dp
    from paper_1801_04380_b200.training import init_parameters
    from oracle.numerics import forward_backward

    ctx = dp.init("gloo")
    net = _net(sn)
    cfg = sn.SimConfig(pool_bytes=1 << 30, features=sn.parse_features(
        "liveness,offload,cache,recompute=cost-aware,convselect"), cost=sn.CostConfig(batch=4))
    rep = sn.run_simulation(net, cfg)
    params = init_parameters(net, seed=2)
    images = torch.randn(8, 3, 32, 32, generator=torch.Generator().manual_seed(0))
    labels = torch.randint(0, 10, (8,), generator=torch.Generator().manual_seed(1))
    shard = slice(4 * rank, 4 * rank + 4)
    _, grads = forward_backward(net, params, images[shard], labels[shard])
    flat = torch.cat([grads[l][k].reshape(-1) for l in sorted(grads) for k in ("w", "b")])
    dp.average_gradients(flat, ctx, scale_in_update=False)
    # numpy payloads are pickled by value (a torch tensor would be shared through
    # a file descriptor that dies with this process)
    out_q.put((rank, flat.numpy().copy(), rep.peak_bytes, rep.pool_high_water_bytes))
    torch.distributed.barrier()
    torch.distributed.destroy_process_group()


def test_two_replicas_equal_full_batch_gradient():
    import sys
    sys.path.insert(0, ROOT)
    import paper_1801_04380_b200 as sn
    from paper_1801_04380_b200.training import init_parameters
    from oracle.numerics import forward_backward

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    results.sort(key=lambda r: r[0])
    (_, g0, peak0, hw0), (_, g1, peak1, hw1) = results
    g0, g1 = torch.from_numpy(g0), torch.from_numpy(g1)
    assert torch.equal(g0, g1)           # every rank holds the same averaged gradient
    assert (peak0, hw0) == (peak1, hw1)  # and planned the identical schedule

    net = _net(sn)
    params = init_parameters(net, seed=2)
    images = torch.randn(8, 3, 32, 32, generator=torch.Generator().manual_seed(0))
    labels = torch.randint(0, 10, (8,), generator=torch.Generator().manual_seed(1))
    _, full = forward_backward(net, params, images, labels)
    ref = torch.cat([full[l][k].reshape(-1) for l in sorted(full) for k in ("w", "b")])
    err = (g0.double() - ref.double()).norm() / ref.double().norm()
    assert err < 1e-5, err


def _bucket_worker(rank: int, world: int, port: int, out_q) -> None:
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    torch.set_num_threads(1)
    import paper_1801_04380_b200 as sn
    from paper_1801_04380_b200 import dp
    from paper_1801_04380_b200.netgen import gen_resnet
    ctx = dp.init("gloo")
    uid = dp.share_unique_id(ctx)  # rank 0's NCCL id, broadcast over gloo
    net = gen_resnet(3, 4, 6, 3)
    cfg = sn.SimConfig(pool_bytes=24 << 30, features=sn.parse_features(
        "liveness,offload,cache,recompute=cost-aware,convselect"), cost=sn.CostConfig(batch=256))
    buckets = dp.bucket_plan(net, cfg, bucket_bytes=4 << 20)
    n = max(hi for _, hi, _ in buckets)
    # stub gradient / parameter blocks standing in for the executor's device blocks
    grads = torch.randn(n, generator=torch.Generator().manual_seed(100 + rank))
    params = torch.randn(n, generator=torch.Generator().manual_seed(7))
    full = grads.clone()
    torch.distributed.all_reduce(full)
    ref = params - 0.01 * (full * (1.0 / world))
    # the executor's order: one all-reduce + update per bucket, in issue order
    for lo, hi, _ in buckets:
        g = grads[lo:hi].clone()
        torch.distributed.all_reduce(g)
        params[lo:hi] -= 0.01 * (g * (1.0 / world))
    out_q.put((rank, uid, buckets, bool(torch.equal(params, ref)), dp.rank_seed(1234, ctx)))
    torch.distributed.barrier()
    torch.distributed.destroy_process_group()


def test_bucketed_allreduce_plumbing_two_ranks():
    """The product's DP host logic at world 2 on gloo: rank 0's NCCL unique id
    reaches every rank; every rank computes the same bucket plan (host only,
    sn_dp_buckets); the buckets are disjoint and cover the parameter block;
    the per-bucket all-reduce + update in issue order equals one global
    all-reduce + SGD bit for bit; ranks draw different dropout seeds."""
    import sys
    sys.path.insert(0, ROOT)
    from oracle.numerics import dropout_keep
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bucket_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(2)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    (_, uid0, b0, ok0, seed0), (_, uid1, b1, ok1, seed1) = res
    assert uid0 == uid1 and len(uid0) == 128
    assert b0 == b1 and len(b0) > 1
    spans = sorted((lo, hi) for lo, hi, _ in b0)
    assert spans[0][0] == 0 and all(a[1] <= b[0] for a, b in zip(spans, spans[1:]))
    assert all(b[0] - a[1] < 64 for a, b in zip(spans, spans[1:]))  # only alignment padding between
    assert ok0 and ok1
    assert seed0 != seed1
    assert not (dropout_keep(4096, 0.5, seed0, 3, 0) == dropout_keep(4096, 0.5, seed1, 3, 0)).all()
