"""SuperNeurons on B200: a memory-scheduled CNN training step.

Drop-in for the reference ``memsched`` API (pkg/src/memsched/__init__.py:69-130):
the network graph, cost model, feature flags and ``run_simulation`` keep their
names and results (bit-identical, via the C++ planner ``libsnplan.so``), and
``run_training`` executes the same schedule for real on a B200 through the
CUDA executor ``libsnexec.so`` (tcgen05/TMEM conv and FC kernels, one
cudaMalloc'd arena at the planner's block offsets, copy-engine offload).
"""

from .convselect import ALGORITHMS, ConvAlgo, Selection, select_algorithm
from .costmodel import (CostConfig, LayerCost, baseline_peak_bytes, build_costs, grad_owner, mib,
                        propagate_shapes)
from .errors import (AllLockedError, ConfigError, CostError, DeviceError, MemschedError, NetError,
                     NetParseError, NetValidationError, PoolError, PoolExhausted, SchedulingError)
from .netgraph import (Layer, LayerKind, NetworkDef, Phase, Schedule, build_schedule,
                       forward_order, load_network, parse_network)
from .simulator import (POLICIES, Features, SimConfig, SimReport, StepRow, SweepPoint,
                        parse_features, run_simulation, run_sweep)
from .analysis import (GradBuffer, LruCache, OffloadPlan, RecomputePlan, Segment, TensorLife,
                       build_offload_plan, demand_peak, grad_buffers, liveness_peak, liveness_table,
                       min_pool_bytes, plan, resident_curve, step_demands, working_set_bytes)
from .netgen import gen_resnet, make_uniform_chain, random_fanjoin
from .poolalloc import BLOCK_BYTES, BlockPool

__version__ = "0.1.0"

__all__ = [
    "ALGORITHMS", "AllLockedError", "BLOCK_BYTES", "BlockPool", "ConfigError", "ConvAlgo", "CostConfig",
    "CostError", "DeviceError", "Features", "GradBuffer", "Layer", "LayerCost", "LayerKind", "LruCache",
    "MemschedError", "NetError", "NetParseError", "NetValidationError", "NetworkDef", "OffloadPlan", "POLICIES",
    "Phase", "PoolError", "PoolExhausted", "RecomputePlan", "Schedule", "SchedulingError", "Segment",
    "Selection", "SimConfig", "SimReport", "StepRow", "SweepPoint", "TensorLife", "baseline_peak_bytes",
    "build_costs", "build_offload_plan", "build_schedule", "demand_peak", "forward_order", "gen_resnet",
    "grad_buffers", "grad_owner", "liveness_peak", "liveness_table", "load_network", "make_uniform_chain", "mib",
    "min_pool_bytes", "parse_features", "parse_network", "plan", "propagate_shapes", "random_fanjoin", "resident_curve",
    "run_simulation", "run_sweep", "select_algorithm", "step_demands", "working_set_bytes", "run_training",
    "__version__",
]


def run_training(*args, **kwargs):
    """Plan like ``run_simulation`` and execute the schedule on a B200 (see training.py)."""
    from .training import run_training as _rt
    return _rt(*args, **kwargs)
