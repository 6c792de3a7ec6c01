"""B200-native Tally: block-level priority scheduling of GPU kernels.

Public API mirrors the reference ``tallysim`` package for the scheduler path
(kernel registration, priority submission, slice/PTB configuration selection
and the scheduler run loop); kernels, launch shapes, preemption and the
real-time dispatch loop are native (``libtally_b200.so``, sm_100a).
"""

__version__ = "0.1.0"

from . import _lib  # noqa: F401  (fails loudly when the native library is missing)
from .device import (BEST_EFFORT, HIGH, B200Device, GpuSpec, KernelCostModel, OriginalShape,
                     PtbShape, SimEvent, SimLaunch, SlicedShape, cost_model, events_to_csv,
                     ms_to_ns, ns_to_ms)
from .profiler import (ConfigCandidate, ProfileKey, ProfileRecord, Profiler, candidate_configs,
                       estimate_turnaround, select_config)
from .scheduler import (EAGER, KERNEL_PRIORITY, POLICIES, TALLY, TIME_SLICED, KernelWork,
                        PolicyRunner, RunResult, SchedulerConfig, TaskScript, run_policy)
from .transforms import TransformError, slice_extents, slice_plan
