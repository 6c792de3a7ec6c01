"""``B200Sim``: the reference ``GpuSim`` surface over the B200, in real time.

The native runner (``csrc/runner.cpp``) drives the B200 through the C++
``CudaDevice``.  Code written against the *reference* surface -- a
``PolicyRunner`` or ``Profiler`` that calls ``submit``, ``signal_preempt``,
``call_at``, ``observer``, ``dispatch_filter``, ``kick``,
``run_to_completion``, ``now`` and ``events`` (ref ``sim.py:229-351``;
consumers ``scheduler.py:183-216``, ``profiler.py:221-236``) -- can drive the
B200 through this class instead, unchanged:

* a ``SimLaunch``'s ``kernel_id`` names a bound ``DeviceKernel``
  (``kernels=`` / :meth:`bind`); its shape picks the launch: ``OriginalShape``
  (a scheduler slice -- fewer blocks than the kernel has -- runs the next
  contiguous range of logical blocks), ``SlicedShape`` (sub-launches strictly
  one after another, ref ``sim.py:447-458``) or ``PtbShape`` (resumable
  persistent workers);
* high-priority launches go to a pool of greatest-priority streams, the rest
  to one least-priority stream per task (their kernels run in order);
* ``signal_preempt`` writes the launch's device flag (a launch not issued yet
  parks at once, ref ``sim.py:344-345``);
* the clock is the host's, in ns since construction; ``call_at`` runs a
  callback at (or, in real time, as soon as possible after) that time;
* ``events`` carries the reference's event kinds: ``LaunchIssued``,
  ``KernelFinished``, ``PreemptSignaled`` and ``WorkerParked`` from the host,
  and ``BlockStarted`` / ``BlockFinished`` per logical block from the
  device's ``%globaltimer`` log (mapped onto the host clock) for the
  streaming and IR-JIT kinds -- the tcgen05 GEMMs do not log blocks.

A parked PTB launch emits one ``WorkerParked`` (the reference emits one per
stopped worker; the runner ticks on the first).
"""

from __future__ import annotations

import heapq

import torch

from . import _lib
from .device import (BLOCK_FINISHED, BLOCK_STARTED, HIGH, KERNEL_FINISHED, LAUNCH_ISSUED,
                     PREEMPT_SIGNALED, WORKER_PARKED, B200Device, SimEvent)
from .kernels import Stream


class B200Handle:
    """KernelHandle fields (ref ``sim.py:175-226``) of one B200 launch."""

    def __init__(self, launch, uid, submit_time):
        self.launch, self.uid, self.submit_time = launch, uid, submit_time
        self.cost, self.shape = launch.cost, launch.shape
        self.ready = self.done = self.parked = self.preempted = False
        self.finish_time = None
        self.preempt_time = None
        self.blocks_finished = 0
        self.sub_completions = []
        self.park_times = []
        self.task_counter = launch.shape.start_count if launch.shape.kind == "ptb" else 0
        self._L = None
        self._sub = 0
        self._offset = 0
        self._log = None
        self._issued = False

    @property
    def is_ptb(self):
        return self.shape.kind == "ptb"

    @property
    def is_sliced(self):
        return self.shape.kind == "sliced"


class B200Sim:
    def __init__(self, gpu=None, placement_seed: int = 0, record_events: bool = True, kernels=None,
                 hp_streams: int = 4, block_events=None):
        self.dev = B200Device.get()
        self.gpu = gpu if gpu is not None else self.dev.spec
        self.record_events = record_events
        self.block_events = record_events if block_events is None else block_events
        self.kernels = dict(kernels or {})
        self.observer = None
        self.dispatch_filter = None
        self.handles = []
        self._events = []
        self._seq = 0
        self._timers, self._tie = [], 0
        self._pending, self._live = [], []
        self._hp = [Stream(True) for _ in range(hp_streams)]
        self._hp_load = [0] * hp_streams
        self._task_streams = {}
        self._slice_next = {}
        self._t0 = B200Device.now_ns()
        self._clk = self.dev.clock_offset()[0]

    def bind(self, kernel_id: str, device_kernel) -> None:
        self.kernels[kernel_id] = device_kernel

    # ---------------------------------------------------------------- clock
    @property
    def now(self) -> int:
        return B200Device.now_ns() - self._t0

    @property
    def events(self):
        return sorted(self._events, key=lambda e: (e.time, e.seq))

    def _emit(self, kind, h, block=-1, t=None):
        ev = SimEvent(self.now if t is None else t, self._seq, kind, h.launch.task_id, h.launch.kernel_id, block)
        self._seq += 1
        if self.record_events:
            self._events.append(ev)
        if self.observer is not None and t is None:
            self.observer(ev)

    def call_at(self, t, fn):
        heapq.heappush(self._timers, (t, self._tie, fn))
        self._tie += 1

    def kick(self):
        self._dispatch()

    # ---------------------------------------------------------------- submit
    def submit(self, launch, at=None) -> B200Handle:
        if launch.kernel_id not in self.kernels:
            raise ValueError(f"{launch.kernel_id}: no device kernel bound")
        if self.gpu.occupancy_limit(launch.cost.threads_per_block) < 1:
            raise ValueError(f"{launch.kernel_id}: block too large for the GPU")
        h = B200Handle(launch, len(self.handles), self.now if at is None else at)
        self.handles.append(h)
        if at is not None and at > self.now:
            self.call_at(at, lambda: self._enqueue(h))
        else:
            self._enqueue(h)
        return h

    def _enqueue(self, h):
        self._pending.append(h)
        self._dispatch()

    def _dispatch(self):
        keep = []
        for hp_pass in (True, False):   # high priority first (ref sim.py:381-393)
            for h in self._pending:
                if (h.launch.priority == HIGH) != hp_pass:
                    continue
                if h.parked:
                    continue
                if self.dispatch_filter is not None and not self.dispatch_filter(h):
                    keep.append(h)
                    continue
                self._issue(h)
        self._pending = keep

    def _stream(self, h):
        if h.launch.priority == HIGH:
            i = min(range(len(self._hp)), key=lambda k: self._hp_load[k])
            self._hp_load[i] += 1
            h._hp_slot = i
            return self._hp[i]
        s = self._task_streams.get(h.launch.task_id)
        if s is None:
            s = self._task_streams[h.launch.task_id] = Stream(False)
        return s

    def _issue(self, h):
        dk = self.kernels[h.launch.kernel_id]
        s = h._stream = self._stream(h)
        total = dk.total_blocks
        if self.block_events:
            h._log = torch.zeros(total, 3, dtype=torch.int64, device="cuda")
        sh = h.shape
        self._emit(LAUNCH_ISSUED, h, -1)
        if sh.kind == "ptb":
            h._L = dk.ptb(s, sh.worker_count, start_count=sh.start_count, block_log=h._log)
        elif sh.kind == "sliced":
            h._L = dk.sliced(s, 0, sh.sub_blocks[0], block_log=h._log)
        elif h.cost.total_blocks != total:
            # a scheduler slice (ref scheduler.py:386-399): the next contiguous range
            key = (h.launch.task_id, h.launch.kernel_id)
            off = self._slice_next.get(key, 0)
            h._offset = off
            h._L = dk.sliced(s, off, h.cost.total_blocks, block_log=h._log)
            self._slice_next[key] = (off + h.cost.total_blocks) % total
        else:
            h._L = dk.original(s, block_log=h._log)
        h._issued = h.ready = True
        self._live.append(h)
        if h.preempted and h.is_ptb:
            h._L.preempt()

    # ---------------------------------------------------------------- preempt
    def signal_preempt(self, h, at=None):
        if not h.is_ptb:
            raise ValueError(f"{h.launch.kernel_id}: not a Ptb launch")
        if h.done:
            raise ValueError(f"{h.launch.kernel_id}: not in flight")
        if at is not None and at > self.now:
            self.call_at(at, lambda: self._preempt(h))
        else:
            self._preempt(h)

    def _preempt(self, h):
        if h.done or h.preempted:
            return
        h.preempted, h.preempt_time = True, self.now
        self._emit(PREEMPT_SIGNALED, h)
        if not h._issued:      # never reached the GPU: parks at once, silently (ref sim.py:338-351)
            h.parked = True
            h.park_times.append(self.now)
            return
        h._L.preempt()

    # ---------------------------------------------------------------- completion
    def _block_events(self, h, base):
        if h._log is None:
            return
        rows = h._log.cpu().tolist()
        off = self._clk - self._t0
        for i, (t0, t1, _who) in enumerate(rows):
            if t1 == 0:
                continue
            b = i - base
            self._emit(BLOCK_STARTED, h, b, t0 + off)
            self._emit(BLOCK_FINISHED, h, b, t1 + off)
            h.blocks_finished += 1
        h._log.zero_()

    def _poll(self) -> bool:
        progress = False
        for h in list(self._live):
            st = h._L.query()
            if not (st.done or st.parked):
                continue
            progress = True
            self._live.remove(h)
            if getattr(h, "_hp_slot", None) is not None:
                self._hp_load[h._hp_slot] -= 1
                h._hp_slot = None
            sh = h.shape
            if sh.kind == "sliced":
                self._block_events(h, 0)
                h.sub_completions.append(self.now)
                h._sub += 1
                if h._sub < len(sh.sub_blocks):
                    off = sum(sh.sub_blocks[:h._sub])
                    self._emit(LAUNCH_ISSUED, h, h._sub)
                    h._L = self.kernels[h.launch.kernel_id].sliced(h._stream, off, sh.sub_blocks[h._sub],
                                                                    block_log=h._log)
                    self._live.append(h)
                    continue
            else:
                self._block_events(h, h._offset if sh.kind == "original" else 0)
            if sh.kind == "ptb":
                h.task_counter = st.task_counter
            if st.parked:
                h.parked = True
                h.park_times.append(self.now)
                self._emit(WORKER_PARKED, h)
            else:
                h.done = True
                h.finish_time = self.now
                self._emit(KERNEL_FINISHED, h)
            self._dispatch()
        return progress

    # ---------------------------------------------------------------- run loop
    def _step(self, until=None):
        while self._timers and self._timers[0][0] <= self.now and (until is None or self._timers[0][0] <= until):
            _t, _k, fn = heapq.heappop(self._timers)
            fn()
        self._poll()
        if self._pending:
            self._dispatch()

    def run_until(self, t):
        if t < self.now:
            raise ValueError(f"cannot run backwards to {t} < now {self.now}")
        start = len(self._events)
        while self.now < t:
            self._step(t)
        return self._events[start:]

    def run_to_completion(self):
        start = len(self._events)
        while self._timers or self._live or any(not h.parked for h in self._pending):
            self._step()
        return self._events[start:]

    def measured_turnaround(self, h, signal_time):
        """ref sim.py:509-526 on the host clock."""
        if h.is_ptb:
            if h.park_times:
                return max(h.park_times) - signal_time
            if h.finish_time is not None:
                return h.finish_time - signal_time
            raise ValueError("no preemption recorded for this launch")
        if h.is_sliced:
            after = [t for t in h.sub_completions if t >= signal_time]
            if not after:
                raise ValueError("no sub-kernel completion after signal time")
            return min(after) - signal_time
        if h.finish_time is None:
            raise ValueError("kernel has not finished")
        return h.finish_time - signal_time

    def close(self):
        for s in self._hp + list(self._task_streams.values()):
            s.close()


def factory(kernels, **kw):
    """A ``sim_cls``-style constructor for runners that build their own
    GpuSim (``factory(kernels)(gpu, placement_seed=..., record_events=...)``)."""
    def make(gpu, placement_seed=0, record_events=True):
        return B200Sim(gpu, placement_seed=placement_seed, record_events=record_events, kernels=kernels, **kw)
    return make


__all__ = ["B200Sim", "B200Handle", "factory"]
_ = _lib
