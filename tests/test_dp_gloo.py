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
