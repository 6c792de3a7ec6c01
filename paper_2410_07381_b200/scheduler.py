"""Priority-aware scheduler: the reference's Python API over the native
policy runner (``csrc/runner.cpp``).

Kernel registration, priority submission and the run loop keep the reference
signatures (ref ``scheduler.py:58-457``):

    KernelWork(kernel_id, cost, exempt=False, kernel=None)
    TaskScript(task_id, priority, kernels, arrivals=())
    SchedulerConfig(policy="Tally", turnaround_threshold_ns=31_600, quantum_ns=2 ms)
    run_policy(gpu, tasks, config, horizon_ns, profiler=None, placement_seed=0,
               record_events=True, device_factory=None) -> RunResult

``kernel=`` binds a :class:`~paper_2410_07381_b200.kernels.DeviceKernel`; with
``device_factory=None`` the run happens in real time on the B200 (the native
dispatch daemon, ``csrc/cuda_device.cpp``).  ``device_factory`` may instead
supply any object with the GpuSim surface (``submit``, ``signal_preempt``,
``call_at``, ``observer``, ``dispatch_filter``, ``kick``,
``run_to_completion``, ``now``, ``events``); the native runner then drives it
through the ``tally_device_vtbl`` callbacks.  The parity tests use that to
show the native runner's dispatch order equals the reference's bit for bit.

Every Tally best-effort kernel's launch configuration comes from
``profiler.select(work.profile_key(), work.cost, threshold)`` exactly as in the
reference (ref ``scheduler.py:371-375``); selections are resolved before the
run starts, which is equivalent because profiling is cached and deterministic.
"""

from __future__ import annotations

import ctypes as C
import sys
from dataclasses import dataclass, field

from . import _lib
from .device import (BEST_EFFORT, EVENT_KINDS, HIGH, KERNEL_FINISHED, WORKER_PARKED, SimEvent,
                     ms_to_ns)
from .profiler import DEFAULT_THRESHOLD_NS, ORIGINAL, PTB, SLICED, ProfileKey, Profiler

TALLY = "Tally"
EAGER = "Eager"
KERNEL_PRIORITY = "KernelPriority"
TIME_SLICED = "TimeSliced"
POLICIES = (TALLY, EAGER, KERNEL_PRIORITY, TIME_SLICED)

DEFAULT_QUANTUM_NS = ms_to_ns(2.0)

INFERENCE = "inference"
TRAINING = "training"


@dataclass(frozen=True)
class SchedulerConfig:
    """ref scheduler.py:58-70."""

    policy: str = TALLY
    turnaround_threshold_ns: int = DEFAULT_THRESHOLD_NS
    quantum_ns: int = DEFAULT_QUANTUM_NS

    def __post_init__(self):
        if self.policy not in POLICIES:
            raise ValueError(f"unknown policy {self.policy!r}")
        if self.turnaround_threshold_ns <= 0:
            raise ValueError("turnaround threshold must be > 0")
        if self.quantum_ns <= 0:
            raise ValueError("time-slice quantum must be > 0")


@dataclass(frozen=True)
class KernelWork:
    """Kernel registration (ref scheduler.py:73-86) + the bound device kernel."""

    kernel_id: str
    cost: object
    exempt: bool = False
    kernel: object = field(default=None, compare=False, repr=False)

    def profile_key(self) -> ProfileKey:
        return ProfileKey(self.kernel_id, (self.cost.total_blocks, 1, 1),
                          (self.cost.threads_per_block, 1, 1))


@dataclass(frozen=True)
class TaskScript:
    """ref scheduler.py:89-112: a kernel pipeline plus traffic (empty arrivals =
    training loop)."""

    task_id: str
    priority: str
    kernels: tuple
    arrivals: tuple = ()

    def __post_init__(self):
        if self.priority not in (HIGH, BEST_EFFORT):
            raise ValueError(f"unknown priority {self.priority!r}")
        if not self.kernels:
            raise ValueError(f"{self.task_id}: empty kernel pipeline")
        if any(b < a for a, b in zip(self.arrivals, self.arrivals[1:])):
            raise ValueError(f"{self.task_id}: arrivals must be non-decreasing")

    @property
    def kind(self) -> str:
        return INFERENCE if self.arrivals else TRAINING


@dataclass
class RunResult:
    """ref scheduler.py:155-161 (+ the B200 per-launch log when run on the device)."""

    events: list
    requests: dict
    iterations: dict
    horizon_ns: int
    launches: list = field(default_factory=list)
    origin_ns: int = 0
    timers: list = field(default_factory=list)   # B200: (scheduled for, fired at) of every runner timer


TIMER_FIRED = 6   # TALLY_EV_TIMER_FIRED: a B200 device-log record, not a reference event kind
_VARIANT_CODE = {ORIGINAL: _lib.SHAPE_ORIGINAL, SLICED: _lib.SHAPE_SLICED, PTB: _lib.SHAPE_PTB}


def _c_cost(cost) -> _lib.c_cost:
    return _lib.c_cost(cost.block_duration_ns, cost.launch_overhead_ns,
                       cost.ptb_iteration_overhead_ns, cost.threads_per_block, cost.total_blocks)


class _ForeignDevice:
    """Adapter: a Python object with the GpuSim surface behind tally_device_vtbl."""

    def __init__(self, sim, runner_id: int):
        self.sim = sim
        self.rid = runner_id
        self.mod = sys.modules[type(sim).__module__]
        self.handles = []
        self.index = {}
        self.error = None
        lib = _lib.lib

        def guard(fn, default=-22):
            def wrapped(*a):
                try:
                    return fn(*a)
                except BaseException as e:   # never unwind through C
                    if self.error is None:
                        self.error = e
                    return default
            return wrapped

        def now(_ctx):
            return self.sim.now

        def submit(_ctx, dp):
            d = dp.contents
            c = d.cost
            cost = self.mod.KernelCostModel(c.block_duration_ns, c.launch_overhead_ns,
                                            c.ptb_iteration_overhead_ns, c.threads_per_block,
                                            c.total_blocks)
            shape = (self.mod.PtbShape(d.worker_count, start_count=d.start_count)
                     if d.shape == _lib.SHAPE_PTB else self.mod.OriginalShape())
            prio = self.mod.HIGH if d.priority == _lib.HIGH_CLASS else self.mod.BEST_EFFORT
            h = self.sim.submit(self.mod.SimLaunch(d.task_id.decode(), d.kernel_id.decode(),
                                                   prio, shape, cost))
            self.index[id(h)] = len(self.handles)
            self.handles.append(h)
            return len(self.handles) - 1

        def preempt(_ctx, h):
            self.sim.signal_preempt(self.handles[h])
            return 0

        def query(_ctx, h, out):
            x = self.handles[h]
            s = out.contents
            s.done, s.parked, s.preempted = int(x.done), int(x.parked), int(x.preempted)
            s.is_ptb = int(x.is_ptb)
            s.task_counter = x.task_counter
            s.finish_time = -1 if x.finish_time is None else x.finish_time
            return 0

        def fire(token):
            def cb():
                rc = lib.tally_runner_fire(self.rid, token)
                if rc < 0:
                    raise _lib.TallyError(f"runner: {_lib.last_error()}")
            return cb

        def call_at(_ctx, t, token):
            self.sim.call_at(t, fire(token))
            return 0

        def dispatch_filter(h):
            rc = lib.tally_runner_filter(self.rid, self.index[id(h)])
            if rc < 0:
                raise _lib.TallyError(f"runner filter: {_lib.last_error()}")
            return rc == 1

        def set_filter(_ctx, enabled):
            self.sim.dispatch_filter = dispatch_filter if enabled else None
            return 0

        def kick(_ctx):
            self.sim.kick()
            return 0

        def run(_ctx):
            self.sim.run_to_completion()
            return 0

        def observe(ev):
            if ev.kind in (KERNEL_FINISHED, WORKER_PARKED):
                rc = lib.tally_runner_on_event(self.rid, EVENT_KINDS.index(ev.kind), 0)
                if rc < 0:
                    raise _lib.TallyError(f"runner: {_lib.last_error()}")

        self.sim.observer = observe
        self._fns = [_lib.NOW_FN(guard(now, 0)), _lib.SUBMIT_FN(guard(submit)),
                     _lib.PREEMPT_FN(guard(preempt)), _lib.QUERY_FN(guard(query)),
                     _lib.CALL_AT_FN(guard(call_at)), _lib.FILTER_FN(guard(set_filter)),
                     _lib.KICK_FN(guard(kick)), _lib.RUN_FN(guard(run))]
        self.vtbl = _lib.c_device_vtbl(None, *self._fns)


class PolicyRunner:
    """Drives one device with one policy over a task set (ref scheduler.py:164-222)."""

    def __init__(self, gpu, tasks, config: SchedulerConfig, horizon_ns: int, profiler=None,
                 placement_seed: int = 0, record_events: bool = True, device_factory=None,
                 options=None):
        if len({t.task_id for t in tasks}) != len(tasks):
            raise ValueError("duplicate task ids")
        self.gpu = gpu
        self.tasks = list(tasks)
        self.config = config
        self.horizon_ns = horizon_ns
        self.placement_seed = placement_seed
        self.record_events = record_events
        self.device_factory = device_factory
        self.options = dict(options or {})
        self.profiler = profiler if profiler is not None else Profiler(
            gpu, device_factory=device_factory)

    def _work(self, work: KernelWork, task: TaskScript) -> _lib.c_work:
        w = _lib.c_work()
        w.kernel_id = work.kernel_id.encode()
        w.cost = _c_cost(work.cost)
        w.exempt = int(work.exempt)
        w.device_kernel = -1 if work.kernel is None else work.kernel.id
        if (self.config.policy == TALLY and task.priority == BEST_EFFORT and not work.exempt):
            if work.kernel is not None and self.device_factory is None:
                self.profiler.bind(work.kernel_id, work.kernel)
            cand = self.profiler.select(work.profile_key(), work.cost,
                                        self.config.turnaround_threshold_ns)
            w.has_config = 1
            w.config.variant = _VARIANT_CODE[cand.variant]
            if cand.fraction is not None:
                w.config.frac_num = cand.fraction.numerator
                w.config.frac_den = cand.fraction.denominator
            w.config.worker_count = cand.worker_count or 0
        if (task.priority == BEST_EFFORT and work.kernel is not None and self.device_factory is None
                and int(self.options.get("lookahead", 1)) > 1):
            # the look-ahead budget: the kernel's untransformed latency (tuner record)
            if self.config.policy != TALLY:
                self.profiler.bind(work.kernel_id, work.kernel)
            w.est_ns = next(r.kernel_latency_ns for r in self.profiler.profile(work.profile_key(), work.cost)
                            if r.candidate.variant == "Original")
        return w

    def run(self) -> RunResult:
        lib = _lib.lib
        rid = C.c_int()
        _lib.check(lib.tally_runner_create(_lib.POLICY_CODES[self.config.policy],
                                           self.config.turnaround_threshold_ns,
                                           self.config.quantum_ns, self.horizon_ns,
                                           C.byref(rid)), "runner")
        rid = rid.value
        try:
            for k, v in self.options.items():
                _lib.check(lib.tally_runner_set_option(rid, k.encode(), int(v)), f"option {k}")
            keep = []
            for t in self.tasks:
                works = (_lib.c_work * len(t.kernels))(*[self._work(w, t) for w in t.kernels])
                arr = (C.c_longlong * max(1, len(t.arrivals)))(*t.arrivals)
                keep.append((works, arr))
                _lib.check(lib.tally_runner_add_task(
                    rid, t.task_id.encode(), _lib.HIGH_CLASS if t.priority == HIGH
                    else _lib.BEST_EFFORT_CLASS, works, len(t.kernels), arr, len(t.arrivals)),
                    "add task")
            if self.device_factory is None:
                return self._run_b200(rid)
            return self._run_foreign(rid)
        finally:
            lib.tally_runner_destroy(rid)

    def _collect(self, rid):
        lib = _lib.lib
        requests, iterations = {}, {}
        for i, t in enumerate(self.tasks):
            n = lib.tally_runner_request_count(rid, i)
            buf = (C.c_longlong * max(1, 2 * n))()
            lib.tally_runner_requests(rid, i, buf, n)
            requests[t.task_id] = [(buf[2 * k], buf[2 * k + 1]) for k in range(n)]
            n = lib.tally_runner_iteration_count(rid, i)
            buf = (C.c_longlong * max(1, n))()
            lib.tally_runner_iterations(rid, i, buf, n)
            iterations[t.task_id] = [buf[k] for k in range(n)]
        return requests, iterations

    def _run_foreign(self, rid) -> RunResult:
        sim = self.device_factory(self.gpu, placement_seed=self.placement_seed,
                                  record_events=self.record_events)
        dev = _ForeignDevice(sim, rid)
        rc = _lib.lib.tally_runner_run(rid, C.byref(dev.vtbl))
        if dev.error is not None:
            raise dev.error
        _lib.check(rc, "runner")
        requests, iterations = self._collect(rid)
        return RunResult(list(sim.events), requests, iterations, self.horizon_ns)

    def _run_b200(self, rid) -> RunResult:
        lib = _lib.lib
        for t in self.tasks:
            for w in t.kernels:
                if w.kernel is None:
                    raise ValueError(f"{w.kernel_id}: KernelWork needs kernel= on the B200")
        _lib.check(lib.tally_runner_run(rid, None), "runner (B200)")
        requests, iterations = self._collect(rid)
        n = lib.tally_device_event_count(rid)
        evs = (_lib.c_event * max(1, n))()
        lib.tally_device_events(rid, evs, n)
        events, timers = [], []
        for k in range(n):
            e = evs[k]
            if e.kind == TIMER_FIRED:
                timers.append((e.block, e.time_ns))   # (scheduled for, ran at)
                continue
            t = self.tasks[e.task]
            kid = t.kernels[e.kernel_index].kernel_id if e.kernel_index >= 0 else "?"
            events.append(SimEvent(e.time_ns, k, EVENT_KINDS[e.kind], t.task_id, kid, e.block))
        n = lib.tally_device_launch_count(rid)
        recs = (_lib.c_launch_record * max(1, n))()
        lib.tally_device_launches(rid, recs, n)
        launches = [{f: getattr(recs[k], f) for f, _ in _lib.c_launch_record._fields_}
                    for k in range(n)]
        return RunResult(events if self.record_events else [], requests, iterations,
                         self.horizon_ns, launches, lib.tally_device_run_origin_ns(rid), timers)


def run_policy(gpu, tasks, config: SchedulerConfig, horizon_ns: int, profiler=None,
               placement_seed: int = 0, record_events: bool = True,
               device_factory=None, options=None) -> RunResult:
    """ref scheduler.py:444-457.  ``options`` (B200 only): {"trace": 1} adds
    GPU-timeline timestamps to ``RunResult.launches``; {"hp_streams": n}."""
    return PolicyRunner(gpu, tasks, config, horizon_ns, profiler=profiler,
                        placement_seed=placement_seed, record_events=record_events,
                        device_factory=device_factory, options=options).run()
