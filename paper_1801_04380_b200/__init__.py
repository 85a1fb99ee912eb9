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

__version__ = "0.1.0"
