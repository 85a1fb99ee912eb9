"""The unified tensor pool's block allocator (drop-in for memsched poolalloc.py).

``BlockPool`` is a thin handle on the planner's C++ pool (``csrc/planner/
pool.cpp``, exported as ``sn_pool_*``): the very allocator whose block offsets
become device-arena addresses in the executor.  Keys may be any hashable; they
are mapped to integer ids on this side.
"""

from __future__ import annotations

import ctypes as C
import io

from . import _cabi
from .errors import PoolError, PoolExhausted

__all__ = ["BLOCK_BYTES", "blocks_for", "BlockPool", "PoolError", "PoolExhausted"]

BLOCK_BYTES = 1024


def blocks_for(nbytes: int) -> int:
    if nbytes < 0:
        raise PoolError(f"negative allocation size {nbytes}")
    return max(1, -(-nbytes // BLOCK_BYTES))


def _lib():
    L = _cabi.lib()
    if not getattr(L, "_sn_pool_cfg", False):
        P = C.POINTER
        L.sn_pool_create.argtypes = [C.c_int64, P(C.c_void_p)]
        L.sn_pool_destroy.argtypes = [C.c_void_p]
        L.sn_pool_destroy.restype = None
        L.sn_pool_alloc.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int32, P(C.c_int64)]
        L.sn_pool_free.argtypes = [C.c_void_p, C.c_int64]
        L.sn_pool_check.argtypes = [C.c_void_p]
        L.sn_pool_stats.argtypes = [C.c_void_p] + [P(C.c_int64)] * 5
        L.sn_pool_spans.argtypes = [C.c_void_p, C.c_int32, P(C.c_int64), P(C.c_int64), P(C.c_int64),
                                    C.c_size_t, P(C.c_size_t)]
        L._sn_pool_cfg = True
    return L


class BlockPool:
    """Fixed-capacity 1 KiB-block arena: first fit from the bottom, or from the
    top of the highest fitting span with ``high=True``; frees coalesce."""

    def __init__(self, capacity_bytes: int) -> None:
        if capacity_bytes < BLOCK_BYTES:
            raise PoolError(f"pool capacity must be at least {BLOCK_BYTES} bytes")
        self._L = _lib()
        self._h = C.c_void_p()
        if self._L.sn_pool_create(int(capacity_bytes), C.byref(self._h)) != 0:
            _cabi.raise_last(self._L)
        self._ids: dict[object, int] = {}
        self._keys: dict[int, object] = {}
        self._next = 0

    def __del__(self) -> None:
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._L.sn_pool_destroy(h)
            self._h = None

    def _stats(self):
        vals = [C.c_int64() for _ in range(5)]
        self._L.sn_pool_stats(self._h, *[C.byref(v) for v in vals])
        return [v.value for v in vals]

    @property
    def capacity_blocks(self) -> int:
        return self._stats()[3]

    @property
    def capacity_bytes(self) -> int:
        return self.capacity_blocks * BLOCK_BYTES

    @property
    def used_bytes(self) -> int:
        return self._stats()[0]

    @property
    def free_bytes(self) -> int:
        return self._stats()[1]

    @property
    def high_water_bytes(self) -> int:
        return self._stats()[2]

    def __contains__(self, key: object) -> bool:
        return key in self._ids

    def __len__(self) -> int:
        return len(self._ids)

    def size_of(self, key: object) -> int:
        kid = self._ids[key]
        for off, length, k in self._spans(False):
            if k == kid:
                return length * BLOCK_BYTES
        raise KeyError(key)

    def alloc(self, key: object, nbytes: int, high: bool = False) -> int:
        if key in self._ids:
            raise PoolError(f"key {key!r} is already allocated")
        blocks_for(nbytes)  # negative sizes -> PoolError
        kid = self._next
        off = C.c_int64()
        if self._L.sn_pool_alloc(self._h, kid, int(nbytes), int(bool(high)), C.byref(off)) != 0:
            _cabi.raise_last(self._L)
        self._next += 1
        self._ids[key] = kid
        self._keys[kid] = key
        return off.value

    def free(self, key: object) -> None:
        if key not in self._ids:
            raise PoolError(f"key {key!r} is not allocated")
        kid = self._ids.pop(key)
        del self._keys[kid]
        if self._L.sn_pool_free(self._h, kid) != 0:
            _cabi.raise_last(self._L)

    def check(self) -> None:
        if self._L.sn_pool_check(self._h) != 0:
            _cabi.raise_last(self._L)

    def _spans(self, free: bool):
        n = C.c_size_t()
        self._L.sn_pool_spans(self._h, int(free), None, None, None, 0, C.byref(n))
        cnt = max(1, n.value)
        offs, lens, keys = (C.c_int64 * cnt)(), (C.c_int64 * cnt)(), (C.c_int64 * cnt)()
        self._L.sn_pool_spans(self._h, int(free), offs, lens, keys, cnt, C.byref(n))
        return [(offs[i], lens[i], keys[i]) for i in range(n.value)]

    def dump(self) -> str:
        used, _, high, cap, _ = self._stats()
        out = io.StringIO()
        out.write(f"pool: {cap} blocks x {BLOCK_BYTES} B, {used // BLOCK_BYTES} used, "
                  f"high water {high // BLOCK_BYTES}\n")
        for off, length, kid in self._spans(False):
            out.write(f"  used  {off:>8} +{length:<8} {self._keys[kid]!r}\n")
        for off, length, _ in self._spans(True):
            out.write(f"  free  {off:>8} +{length:<8}\n")
        return out.getvalue()
