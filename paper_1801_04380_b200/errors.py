"""Exception taxonomy of the drop-in API.

Mirrors the reference hierarchy (memsched errors.py:8-17 plus the subclasses
declared next to their modules: netgraph.py:19-32, costmodel.py:23-24,
poolalloc.py:21-26, offload.py:21-22), so ``except memsched.X`` handlers keep
working.  The CLI convention is unchanged: SchedulingError -> exit 3, any other
MemschedError -> exit 2.  ``DeviceError`` is new: the B200 executor failed
(CUDA/NCCL), which the simulator could never do.
"""

from __future__ import annotations


class MemschedError(Exception):
    """Root of every error raised by the scheduler API."""


class ConfigError(MemschedError):
    """The run configuration is rejected (flags, values, pool below the floor)."""


class SchedulingError(MemschedError):
    """The schedule cannot be executed in the configured pool."""


class NetError(MemschedError):
    """A network definition problem."""


class NetParseError(NetError):
    """Malformed network text; ``lineno`` is the 1-based offending line."""

    def __init__(self, message: str, lineno: int) -> None:
        super().__init__(f"line {lineno}: {message}")
        self.lineno = lineno


class NetValidationError(NetError):
    """The layer graph violates a structural rule."""


class CostError(MemschedError):
    """Layer parameters or input shapes admit no cost."""


class PoolError(MemschedError):
    """Block-pool misuse: duplicate/unknown keys, bad sizes, corrupted spans."""


class PoolExhausted(SchedulingError):
    """No free span can hold the requested allocation."""


class AllLockedError(SchedulingError):
    """Eviction was needed but no cached tensor can be evicted."""


class DeviceError(MemschedError):
    """The B200 executor hit a CUDA / NCCL failure or an unsupported graph."""


# sn_error_kind (include/superneurons.h) -> exception class
KIND_TO_EXC = {
    1: ConfigError,
    2: SchedulingError,
    3: CostError,
    4: NetValidationError,
    5: PoolError,
    6: PoolExhausted,
    7: AllLockedError,
    8: ZeroDivisionError,
    9: MemschedError,
    10: DeviceError,
    11: DeviceError,
}
