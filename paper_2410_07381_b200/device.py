"""The device boundary: value types of the reference GpuSim surface plus the
B200 device binding.

Types mirror ``tallysim.sim`` (ref ``sim.py:24-172``) so that code written
against the reference keeps working: ``GpuSpec``, ``KernelCostModel``,
``cost_model``, the three launch shapes, ``SimLaunch``, ``SimEvent`` and
``events_to_csv``.  ``B200Device`` binds libtally_b200 to one GPU and reports
its real ``GpuSpec``; the real-time run loop itself is native
(``csrc/cuda_device.cpp``) and is entered through
``scheduler.run_policy(..., device=None)``.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _lib

NS_PER_US = 1_000
NS_PER_MS = 1_000_000
NS_PER_S = 1_000_000_000

HIGH = "High"
BEST_EFFORT = "BestEffort"

LAUNCH_ISSUED = "LaunchIssued"
BLOCK_STARTED = "BlockStarted"
BLOCK_FINISHED = "BlockFinished"
KERNEL_FINISHED = "KernelFinished"
PREEMPT_SIGNALED = "PreemptSignaled"
WORKER_PARKED = "WorkerParked"
EVENT_KINDS = (LAUNCH_ISSUED, BLOCK_STARTED, BLOCK_FINISHED, KERNEL_FINISHED,
               PREEMPT_SIGNALED, WORKER_PARKED)          # index = TALLY_EV_* code

DEFAULT_LAUNCH_OVERHEAD_NS = 5 * NS_PER_US


def ms_to_ns(ms: float) -> int:
    """ref sim.py:29-30 (Python round: half-even)."""
    return round(ms * NS_PER_MS)


def ns_to_ms(ns: int) -> float:
    return ns / NS_PER_MS


def default_ptb_iteration_overhead_ns(block_duration_ns: int) -> int:
    """ref sim.py:51-52."""
    return block_duration_ns // 50 + NS_PER_US


@dataclass(frozen=True)
class GpuSpec:
    """ref sim.py:55-74."""

    num_sms: int
    max_threads_per_sm: int
    max_blocks_per_sm: int

    def __post_init__(self):
        if min(self.num_sms, self.max_threads_per_sm, self.max_blocks_per_sm) < 1:
            raise ValueError(f"all GpuSpec fields must be >= 1: {self}")

    def occupancy_limit(self, threads_per_block: int) -> int:
        if threads_per_block < 1:
            raise ValueError("threads_per_block must be >= 1")
        return min(self.max_blocks_per_sm, self.max_threads_per_sm // threads_per_block)

    @property
    def total_slots(self) -> int:
        return self.num_sms * self.max_blocks_per_sm


@dataclass(frozen=True)
class KernelCostModel:
    """ref sim.py:77-90.  On the B200 the durations are *measured* per kernel
    (PAPER.md:232); the scheduler itself only consumes ``total_blocks`` and
    ``threads_per_block``."""

    block_duration_ns: int
    launch_overhead_ns: int
    ptb_iteration_overhead_ns: int
    threads_per_block: int
    total_blocks: int

    def __post_init__(self):
        if min(self.block_duration_ns, self.launch_overhead_ns,
               self.ptb_iteration_overhead_ns) < 0:
            raise ValueError("durations must be non-negative")
        if self.total_blocks < 1 or self.threads_per_block < 1:
            raise ValueError("block counts must be >= 1")


def cost_model(block_duration_ms, total_blocks, threads_per_block=32,
               launch_overhead_ms=None, ptb_iteration_overhead_ms=None) -> KernelCostModel:
    """ref sim.py:93-111."""
    d = ms_to_ns(block_duration_ms)
    lo = DEFAULT_LAUNCH_OVERHEAD_NS if launch_overhead_ms is None else ms_to_ns(launch_overhead_ms)
    it = (default_ptb_iteration_overhead_ns(d) if ptb_iteration_overhead_ms is None
          else ms_to_ns(ptb_iteration_overhead_ms))
    return KernelCostModel(d, lo, it, threads_per_block, total_blocks)


@dataclass(frozen=True)
class OriginalShape:
    kind = "original"


@dataclass(frozen=True)
class SlicedShape:
    sub_blocks: tuple
    kind = "sliced"

    def __post_init__(self):
        if not self.sub_blocks or min(self.sub_blocks) < 1:
            raise ValueError("sub-launch block counts must be >= 1")


@dataclass(frozen=True)
class PtbShape:
    worker_count: int
    start_count: int = 0
    kind = "ptb"

    def __post_init__(self):
        if self.worker_count < 1:
            raise ValueError("worker count must be >= 1")
        if self.start_count < 0:
            raise ValueError("persisted counter must be >= 0")


@dataclass(frozen=True)
class SimLaunch:
    """Priority submission record (ref sim.py:140-153)."""

    task_id: str
    kernel_id: str
    priority: str
    shape: object
    cost: KernelCostModel

    def __post_init__(self):
        if self.priority not in (HIGH, BEST_EFFORT):
            raise ValueError(f"unknown priority {self.priority!r}")
        if self.shape.kind == "sliced" and sum(self.shape.sub_blocks) != self.cost.total_blocks:
            raise ValueError("sliced sub-launch blocks must sum to total_blocks")


@dataclass(frozen=True)
class SimEvent:
    """ref sim.py:156-166."""

    time: int
    seq: int
    kind: str
    task: str
    kernel: str
    block: int

    def csv_row(self) -> str:
        return f"{self.time},{self.kind},{self.task},{self.kernel},{self.block}"


def events_to_csv(events) -> str:
    """ref sim.py:169-172: ``time_ns,kind,task,kernel,block``."""
    return "time_ns,kind,task,kernel,block\n" + "".join(e.csv_row() + "\n" for e in events)


class B200Device:
    """One B200 bound to libtally_b200 (ref ``GpuSim(gpu)`` construction).

    ``spec`` is the device's real ``GpuSpec`` (148 SMs, 2048 threads, 32
    blocks per SM on a B200).  Idempotent per process: constructing it twice
    for the same ordinal returns the same binding.
    """

    _bound: dict = {}

    def __init__(self, device: int = 0):
        info = _lib.c_gpu_info()
        _lib.check(_lib.lib.tally_init(device, C.byref(info)), "tally_init")
        self.info = info
        self.device = device
        self.name = info.name.decode()
        self.spec = GpuSpec(info.num_sms, info.max_threads_per_sm, info.max_blocks_per_sm)
        self.stream_mem_ops = bool(info.stream_mem_ops)
        B200Device._bound[device] = self

    @classmethod
    def get(cls, device: int = 0) -> "B200Device":
        return cls._bound.get(device) or cls(device)

    def set_flag_mode(self, host_mapped: bool):
        """Where PTB preemption flags live: device memory written with
        cuStreamWriteValue32 (default) or mapped pinned host memory."""
        _lib.check(_lib.lib.tally_set_flag_mode(1 if host_mapped else 0), "flag mode")

    def clock_offset(self):
        """(host_ns - device_globaltimer_ns, uncertainty_ns)."""
        off, unc = C.c_longlong(), C.c_longlong()
        _lib.check(_lib.lib.tally_clock_offset(C.byref(off), C.byref(unc)), "clock offset")
        return off.value, unc.value

    @staticmethod
    def now_ns() -> int:
        return _lib.lib.tally_now_ns()
