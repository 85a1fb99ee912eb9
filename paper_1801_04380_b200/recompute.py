"""Reference module layout: ``memsched.recompute`` (pkg/src/memsched/recompute.py).

The implementations live in ``analysis.py``; this module keeps the
reference's import path for drop-in callers."""

from .analysis import (POLICIES, DemandPeak, RecomputePlan, Segment, build_segments, demand_peak,  # noqa: F401
                       first_backward_use, memory_extras, min_pool_bytes, plan, speed_extras, speed_prediction,
                       step_demands)
