"""Reference module layout: ``memsched.offload`` (pkg/src/memsched/offload.py).

The implementations live in ``analysis.py``; this module keeps the
reference's import path for drop-in callers."""

from .analysis import (OFFLOAD_KINDS, LruCache, OffloadPlan, build_offload_plan,  # noqa: F401
                       offload_candidates)
from .errors import AllLockedError  # noqa: F401
