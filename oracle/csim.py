"""GpuSim surface over the C restatement of the reference GPU (``csim.c``).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``): the same contract as
``oracle.gpu_model.GpuSim`` (ref ``sim.py:229-526``) -- ``submit``,
``signal_preempt``, ``call_at``, ``observer``, ``dispatch_filter``, ``kick``,
``run_until``, ``run_to_completion``, ``now``, ``events`` and the handle
fields -- with the event loop in C.  ``tests/test_oracle_csim.py`` requires it
to reproduce the reference's golden event logs byte for byte; ``bench.py``'s
CPU reference arm uses it so that a B200-scale co-location window (millions of
logical blocks) simulates in seconds.

The SM placement order is drawn here with CPython's ``random.Random``
(ref ``sim.py:247-249``) and handed to C as data.
"""

from __future__ import annotations

import ctypes as C
import os
import random
import subprocess

from .gpu_model import (BEST_EFFORT, BLOCK_FINISHED, BLOCK_STARTED, HIGH, KERNEL_FINISHED,
                        LAUNCH_ISSUED, PREEMPT_SIGNALED, WORKER_PARKED, SimEvent)

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csim.c")
LIB = os.path.join(HERE, "_build", "libcsim.so")
KINDS = (LAUNCH_ISSUED, BLOCK_STARTED, BLOCK_FINISHED, KERNEL_FINISHED, PREEMPT_SIGNALED, WORKER_PARKED)
_KIND_BIT = {k: 1 << i for i, k in enumerate(KINDS)}
_SHAPE = {"original": 0, "sliced": 1, "ptb": 2}


def build(force=False):
    """Compile csim.c into oracle/_build/libcsim.so (gcc, seconds)."""
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    tmp = LIB + f".{os.getpid()}.tmp"
    subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", tmp, SRC])
    os.replace(tmp, LIB)
    return LIB


class _Handle(C.Structure):
    _fields_ = [(n, C.c_longlong) for n in (
        "uid", "priority", "shape", "block_ns", "launch_ns", "iter_ns", "tpb", "total",
        "worker_count", "start_count", "ready", "done", "preempted", "parked",
        "finish_time", "preempt_time", "blocks_finished", "next_block", "current_sub",
        "sub_placed", "sub_finished", "task_counter", "workers_placed", "workers_active",
        "submit_time", "n_sub", "n_sub_completions", "n_park_times")]


class _Event(C.Structure):
    _fields_ = [(n, C.c_longlong) for n in ("time", "seq", "kind", "uid", "block")]


_OBS = C.CFUNCTYPE(None, C.c_longlong, C.c_longlong, C.c_longlong, C.c_longlong)
_FILT = C.CFUNCTYPE(C.c_int, C.c_longlong)
_CB = C.CFUNCTYPE(None, C.c_longlong)
_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        P, ll = C.c_void_p, C.c_longlong
        L.csim_new.restype = P
        L.csim_new.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), C.c_int]
        L.csim_free.argtypes = [P]
        L.csim_set_callbacks.argtypes = [P, _OBS, C.c_uint, _FILT, _CB]
        L.csim_abort.argtypes = [P]
        for f in ("csim_now", "csim_nlogged", "csim_nevents", "csim_pending"):
            getattr(L, f).restype = ll
            getattr(L, f).argtypes = [P]
        L.csim_events.restype = C.POINTER(_Event)
        L.csim_events.argtypes = [P]
        L.csim_call_at.argtypes = [P, ll, ll]
        L.csim_submit.restype = ll
        L.csim_submit.argtypes = [P] + [ll] * 10 + [C.POINTER(ll), ll]
        L.csim_handle.restype = C.POINTER(_Handle)
        L.csim_handle.argtypes = [P, ll]
        L.csim_sub_completions.restype = C.POINTER(ll)
        L.csim_sub_completions.argtypes = [P, ll]
        L.csim_park_times.restype = C.POINTER(ll)
        L.csim_park_times.argtypes = [P, ll]
        L.csim_signal_preempt.argtypes = [P, ll, ll]
        L.csim_kick.argtypes = [P]
        L.csim_run.restype = C.c_int
        L.csim_run.argtypes = [P, ll, C.c_int]
        _lib = L
    return _lib


class KernelHandle:
    """Per-launch state (ref ``sim.py:175-226``), read live from the C record."""

    __slots__ = ("launch", "uid", "cost", "shape", "_r", "_sim")

    def __init__(self, sim, launch, uid):
        self._sim, self.launch, self.uid = sim, launch, uid
        self.cost, self.shape = launch.cost, launch.shape
        self._r = lib().csim_handle(sim._s, uid).contents

    is_ptb = property(lambda self: self.shape.kind == "ptb")
    is_sliced = property(lambda self: self.shape.kind == "sliced")
    submit_time = property(lambda self: self._r.submit_time)
    ready = property(lambda self: bool(self._r.ready))
    done = property(lambda self: bool(self._r.done))
    preempted = property(lambda self: bool(self._r.preempted))
    parked = property(lambda self: bool(self._r.parked))
    task_counter = property(lambda self: self._r.task_counter)
    blocks_finished = property(lambda self: self._r.blocks_finished)
    workers_placed = property(lambda self: self._r.workers_placed)
    workers_active = property(lambda self: self._r.workers_active)
    next_block = property(lambda self: self._r.next_block)
    current_sub = property(lambda self: self._r.current_sub)

    @property
    def finish_time(self):
        t = self._r.finish_time
        return None if t < 0 else t

    @property
    def preempt_time(self):
        t = self._r.preempt_time
        return None if t < 0 else t

    @property
    def sub_completions(self):
        n = self._r.n_sub_completions
        p = lib().csim_sub_completions(self._sim._s, self.uid)
        return [p[i] for i in range(n)]

    @property
    def park_times(self):
        n = self._r.n_park_times
        p = lib().csim_park_times(self._sim._s, self.uid)
        return [p[i] for i in range(n)]

    def unplaced_blocks(self):
        r = self._r
        if r.done or r.parked:
            return 0
        if self.is_ptb:
            return 0 if r.preempted else r.worker_count - r.workers_placed
        if self.is_sliced:
            subs = self.shape.sub_blocks
            return subs[r.current_sub] - r.sub_placed + sum(subs[r.current_sub + 1:])
        return r.total - r.next_block


class _EventsSince:
    """The events a run logged (``sim.py`` returns ``events[start:]``),
    converted to SimEvents only when read: the profiler ignores them, and
    materialising millions of records would cost more than simulating them."""

    def __init__(self, sim, start):
        self._sim, self._start, self._stop = sim, start, lib().csim_nevents(sim._s)

    def _list(self):
        return self._sim.events[self._start:self._stop]

    def __len__(self):
        return self._stop - self._start

    def __iter__(self):
        return iter(self._list())

    def __getitem__(self, i):
        return self._list()[i]

    def __eq__(self, other):
        return self._list() == list(other)

    def __repr__(self):
        return repr(self._list())


class GpuSim:
    """``oracle.gpu_model.GpuSim`` with the event loop in C."""

    def __init__(self, gpu, placement_seed: int = 0, record_events: bool = True):
        self.gpu = gpu
        self.record_events = record_events
        order = list(range(gpu.num_sms))
        random.Random(placement_seed).shuffle(order)
        self._sm_order = order
        L = lib()
        self._s = L.csim_new(gpu.num_sms, gpu.max_threads_per_sm, gpu.max_blocks_per_sm,
                             (C.c_int * gpu.num_sms)(*order), 1 if record_events else 0)
        self.handles = []
        self._fns = {}
        self._next_tok = 0
        self._observer = None
        self._observe_mask = (1 << len(KINDS)) - 1
        self._filter = None
        self._exc = None
        self._events = []
        # ctypes callbacks (kept referenced for the sim's lifetime)
        self._c_obs = _OBS(self._on_obs)
        self._c_filt = _FILT(self._on_filt)
        self._c_cb = _CB(self._on_cb)
        self._c_none_obs = C.cast(None, _OBS)
        self._c_none_filt = C.cast(None, _FILT)
        self._install()

    def __del__(self):
        s = getattr(self, "_s", None)
        if s:
            lib().csim_free(s)
            self._s = None

    # callback plumbing -------------------------------------------------------
    def _install(self):
        lib().csim_set_callbacks(self._s, self._c_obs if self._observer else self._c_none_obs,
                                 self._observe_mask, self._c_filt if self._filter else self._c_none_filt,
                                 self._c_cb)

    def _fail(self, e):
        if self._exc is None:
            self._exc = e
        lib().csim_abort(self._s)

    def _on_obs(self, kind, uid, block, seq):
        if self._exc is not None:
            return
        try:
            h = self.handles[uid]
            self._observer(SimEvent(self.now, seq, KINDS[kind], h.launch.task_id, h.launch.kernel_id, block))
        except BaseException as e:    # noqa: BLE001 -- re-raised by the run loop
            self._fail(e)

    def _on_filt(self, uid):
        if self._exc is not None:
            return 1
        try:
            return 1 if self._filter(self.handles[uid]) else 0
        except BaseException as e:    # noqa: BLE001
            self._fail(e)
            return 1

    def _on_cb(self, tok):
        if self._exc is not None:
            return
        try:
            self._fns.pop(tok)()
        except BaseException as e:    # noqa: BLE001
            self._fail(e)

    @property
    def observer(self):
        return self._observer

    @observer.setter
    def observer(self, fn):
        self._observer = fn
        self._install()

    def observe_kinds(self, kinds):
        """Deliver only these event kinds to the observer (a consumer that
        ignores the others, like the policy runner, sees identical behaviour)."""
        self._observe_mask = sum(_KIND_BIT[k] for k in kinds)
        self._install()

    @property
    def dispatch_filter(self):
        return self._filter

    @dispatch_filter.setter
    def dispatch_filter(self, fn):
        self._filter = fn
        self._install()

    # clock and log -----------------------------------------------------------
    @property
    def now(self):
        return lib().csim_now(self._s)

    @property
    def _nlogged(self):
        return lib().csim_nlogged(self._s)

    @property
    def events(self):
        L = lib()
        n = L.csim_nevents(self._s)
        if len(self._events) < n:
            p = L.csim_events(self._s)
            hs = self.handles
            for i in range(len(self._events), n):
                e = p[i]
                h = hs[e.uid]
                self._events.append(SimEvent(e.time, e.seq, KINDS[e.kind], h.launch.task_id,
                                             h.launch.kernel_id, e.block))
        return self._events

    def _run(self, until, bounded):
        rc = lib().csim_run(self._s, until, 1 if bounded else 0)
        if self._exc is not None:
            e, self._exc = self._exc, None
            raise e
        if rc != 0:
            raise RuntimeError("csim run aborted")

    def call_at(self, t, fn):
        if t < self.now:
            raise ValueError(f"cannot schedule at {t} < now {self.now}")
        tok = self._next_tok
        self._next_tok += 1
        self._fns[tok] = fn
        lib().csim_call_at(self._s, t, tok)

    def run_until(self, t):
        if t < self.now:
            raise ValueError(f"cannot run backwards to {t} < now {self.now}")
        start = lib().csim_nevents(self._s)
        self._run(t, True)
        return _EventsSince(self, start)

    def run_to_completion(self):
        start = lib().csim_nevents(self._s)
        self._run(0, False)
        return _EventsSince(self, start)

    def kick(self):
        lib().csim_kick(self._s)
        if self._exc is not None:
            e, self._exc = self._exc, None
            raise e

    # submission --------------------------------------------------------------
    def submit(self, launch, at=None):
        now = self.now
        at = now if at is None else at
        if at < now:
            raise ValueError(f"cannot submit at {at} < now {now}")
        if self.gpu.occupancy_limit(launch.cost.threads_per_block) < 1:
            raise ValueError(f"{launch.kernel_id}: block too large for the GPU")
        c, sh = launch.cost, launch.shape
        kind = _SHAPE[sh.kind]
        subs = sh.sub_blocks if sh.kind == "sliced" else ()
        arr = (C.c_longlong * max(1, len(subs)))(*subs)
        uid = lib().csim_submit(self._s, at, 0 if launch.priority == HIGH else 1, kind, c.block_duration_ns,
                                c.launch_overhead_ns, c.ptb_iteration_overhead_ns, c.threads_per_block,
                                c.total_blocks, sh.worker_count if kind == 2 else 0,
                                sh.start_count if kind == 2 else 0, arr, len(subs))
        h = KernelHandle(self, launch, uid)
        self.handles.append(h)
        return h

    def signal_preempt(self, h, at=None):
        if not h.is_ptb:
            raise ValueError(f"{h.launch.kernel_id}: not a Ptb launch")
        if h.done:
            raise ValueError(f"{h.launch.kernel_id}: not in flight")
        lib().csim_signal_preempt(self._s, h.uid, self.now if at is None else at)

    def measured_turnaround(self, h, signal_time):
        if h.is_ptb:
            pt = h.park_times
            if pt:
                return max(pt) - signal_time
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


__all__ = ["GpuSim", "KernelHandle", "build", "HIGH", "BEST_EFFORT"]
