"""Reference module layout: ``memsched.liveness`` (pkg/src/memsched/liveness.py).

The implementations live in ``analysis.py`` (over the C++ planner's tables);
this module keeps the reference's import path for drop-in callers."""

from .analysis import (GradBuffer, TensorLife, backward_use_steps, curve_peak, dump_liveness_csv,  # noqa: F401
                       forward_use_steps, grad_buffers, last_forward_use_step, last_use_step, liveness_peak,
                       liveness_table, resident_curve, working_set_bytes)
