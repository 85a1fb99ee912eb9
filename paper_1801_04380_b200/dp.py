"""Data-parallel replicas: one process per GPU, the weight gradients summed by
NCCL inside the executor (the only collective of the path).

Every rank plans the identical schedule (the plan depends only on the net,
per-replica batch, pool and features -- parameters and their gradients live
outside the pool accounting, reference costmodel.py:3-6), so the collective
cannot perturb residency.  The executor (``Executor(..., dp=ctx)``) sums the
gradients in buckets with ``ncclAllReduce`` on its own communication stream,
each bucket issued as soon as the backward steps of its layers are done, and
applies ``lr * grad / world`` per bucket right after its all-reduce -- no host
synchronisation inside a step.  The communicator is created from an NCCL
unique id that rank 0 makes and the torch.distributed group (gloo or nccl)
broadcasts.  Weights start identical on every rank (same init seed);
``broadcast_parameters`` exists for externally supplied weights.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

__all__ = ["DPContext", "init", "rank_seed", "unique_id", "share_unique_id", "bucket_plan", "nccl_version",
           "average_gradients", "broadcast_parameters"]


class DPIdC(C.Structure):
    _fields_ = [("bytes", C.c_ubyte * 128)]  # c_ubyte: a c_char field would stop at the first NUL


def _lib():
    from . import _native
    L = _native.executor()
    if not getattr(L, "_sn_dp_configured", False):
        L.sn_dp_last_error.restype = C.c_char_p
        L.sn_dp_nccl_version.argtypes = [C.POINTER(C.c_int32)]
        L.sn_dp_unique_id.argtypes = [C.POINTER(DPIdC)]
        L.sn_dp_comm_create.argtypes = [C.POINTER(DPIdC), C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]
        L.sn_dp_comm_destroy.argtypes = [C.c_void_p]
        L.sn_dp_comm_destroy.restype = None
        L.sn_dp_buckets.argtypes = [C.c_void_p, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                    C.POINTER(C.c_int32), C.c_size_t, C.POINTER(C.c_size_t)]
        L._sn_dp_configured = True
    return L


def _err(L) -> str:
    return L.sn_dp_last_error().decode("utf-8", "replace")


@dataclass
class DPContext:
    rank: int = 0
    world: int = 1
    local_rank: int = 0
    backend: str = "none"
    force_comm: bool = False  # build a communicator even at world 1 (tests the DP program path)
    _comm: int | None = field(default=None, repr=False)
    _uid: bytes | None = field(default=None, repr=False)

    @property
    def active(self) -> bool:
        return self.world > 1

    def comm(self, device: int) -> int:
        """The NCCL communicator of this rank (created on first use)."""
        if self._comm is None:
            L = _lib()
            uid = self._uid if self._uid is not None else share_unique_id(self)
            cid = DPIdC()
            C.memmove(C.addressof(cid), uid, 128)
            out = C.c_void_p()
            if L.sn_dp_comm_create(C.byref(cid), self.world, self.rank, device, C.byref(out)) != 0:
                from .errors import DeviceError
                raise DeviceError(_err(L))
            self._comm = out.value
        return self._comm

    def close(self) -> None:
        if self._comm is not None:
            _lib().sn_dp_comm_destroy(self._comm)
            self._comm = None


def init(backend: str | None = None) -> DPContext:
    """Initialise from torchrun's environment (RANK/WORLD_SIZE/LOCAL_RANK)."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world <= 1:
        return DPContext()
    if backend is None:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
    if not dist.is_initialized():
        kw = {}
        if backend == "nccl":
            torch.cuda.set_device(local)
            kw["device_id"] = torch.device(f"cuda:{local}")
        dist.init_process_group(backend, **kw)
    return DPContext(rank=rank, world=world, local_rank=local, backend=backend)


def rank_seed(base: int, ctx: DPContext) -> int:
    """Per-rank seed (data shards, dropout masks): replicas must not draw the
    same masks on their local batches, or the step is not a global-batch step."""
    return base + 7919 * ctx.rank


def nccl_version() -> int:
    L = _lib()
    v = C.c_int32()
    if L.sn_dp_nccl_version(C.byref(v)) != 0:
        from .errors import DeviceError
        raise DeviceError(_err(L))
    return v.value


def unique_id() -> bytes:
    """A fresh NCCL unique id (rank 0)."""
    L = _lib()
    out = DPIdC()
    if L.sn_dp_unique_id(C.byref(out)) != 0:
        from .errors import DeviceError
        raise DeviceError(_err(L))
    return C.string_at(C.addressof(out), 128)


def share_unique_id(ctx: DPContext) -> bytes:
    """Rank 0 makes the NCCL id; the torch.distributed group broadcasts it."""
    import torch
    if not ctx.active:
        uid = unique_id()
    else:
        import torch.distributed as dist
        dev = f"cuda:{ctx.local_rank}" if ctx.backend == "nccl" else "cpu"
        buf = torch.zeros(128, dtype=torch.uint8, device=dev)
        if ctx.rank == 0:
            buf.copy_(torch.frombuffer(bytearray(unique_id()), dtype=torch.uint8))
        dist.broadcast(buf, 0)
        uid = bytes(buf.cpu().tolist())
    ctx._uid = uid
    return uid


def bucket_plan(net, config, bucket_bytes: int = 0) -> list[tuple[int, int, int]]:
    """(lo, hi, after_layer) of every all-reduce bucket, in issue order --
    the executor's own plan, computed on the host (no device needed)."""
    from .simulator import plan_handle
    L = _lib()
    h = plan_handle(net, config)
    n = C.c_size_t()
    if L.sn_dp_buckets(h.ptr, bucket_bytes, None, None, None, 0, C.byref(n)) != 0:
        raise RuntimeError(_native_err())
    lo, hi = (C.c_int64 * max(1, n.value))(), (C.c_int64 * max(1, n.value))()
    after = (C.c_int32 * max(1, n.value))()
    if L.sn_dp_buckets(h.ptr, bucket_bytes, lo, hi, after, n.value, C.byref(n)) != 0:
        raise RuntimeError(_native_err())
    return [(lo[i], hi[i], after[i]) for i in range(n.value)]


def _native_err() -> str:
    L = _lib()
    L.sn_exec_last_error.restype = C.c_char_p
    return L.sn_exec_last_error().decode("utf-8", "replace")


def average_gradients(flat, ctx: DPContext, scale_in_update: bool = True):
    """Sum a flat fp32 gradient block over ranks through torch.distributed (for
    external training loops; the executor's own DP path does this in NCCL
    buckets inside the step)."""
    if not ctx.active:
        return flat
    import torch.distributed as dist
    dist.all_reduce(flat, op=dist.ReduceOp.SUM)
    if not scale_in_update:
        flat.div_(ctx.world)
    return flat


def broadcast_parameters(flat, ctx: DPContext, src: int = 0):
    if ctx.active:
        import torch.distributed as dist
        dist.broadcast(flat, src)
    return flat
