"""Replay a B200 run's observed outcomes through the oracle policy runner.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  Dispatch-order
parity is defined in virtual time: the scheduler is a pure
function of (arrivals, the order and outcome of kernel completions and
parkings).  On the B200 the native runner's decisions are logged
(``RunResult.launches``: every submission with its shape, workers and resume
counter, and the host time it completed or parked).  ``ReplaySim`` is a
GpuSim-surface device that, when the reference runner (``oracle.policy``,
ref ``scheduler.py:164-441``) submits a launch, completes it at the B200's
recorded time with the B200's recorded outcome; the arrivals are the same.
If the reference runner then submits exactly the launches the B200 runner
did, in the same order, and preempts the same ones, the B200 dispatch order
equals the reference's on that trace.
"""

from __future__ import annotations

import heapq
from collections import deque

from .gpu_model import KERNEL_FINISHED, PREEMPT_SIGNALED, WORKER_PARKED, SimEvent
from .tuner import ConfigCandidate

_SHAPES = {0: "original", 1: "original", 2: "ptb"}   # a B200 slice is an Original launch of `count` blocks


class _Handle:
    def __init__(self, launch, rec):
        self.launch, self.rec = launch, rec
        self.cost, self.shape = launch.cost, launch.shape
        self.done = self.parked = self.preempted = False
        self.task_counter = launch.shape.start_count if launch.shape.kind == "ptb" else 0
        self.finish_time = None
        self.sub_completions = []

    @property
    def is_ptb(self):
        return self.shape.kind == "ptb"


class ReplaySim:
    """GpuSim surface (ref sim.py:229-351) whose launches finish when and how
    the B200 run's did.  ``records``: the B200 ``RunResult.launches`` dicts;
    ``names``: (task index, kernel index) -> (task_id, kernel_id)."""

    def __init__(self, records, names, timers=()):
        self.now = 0
        # runner timers run when the B200 daemon ran them (an arrival meets a
        # completion in the order the daemon saw them, not in trace order)
        self._fired = {}
        for t, f in timers:
            self._fired.setdefault(t, []).append(f)
        self._q, self._tie = [], 0
        self.observer = None
        self.dispatch_filter = None
        self.events = []
        self._seq = 0
        self.expected = deque(sorted(records, key=lambda r: r["handle"]))
        self.names = names
        self.submitted = []     # (task_id, kernel_id, shape, workers, start, blocks) in order
        self.preempts = []      # (task_id, kernel_id, start) in order
        self.mismatch = None

    def _at(self, t, fn):
        heapq.heappush(self._q, (t, self._tie, fn))
        self._tie += 1

    def call_at(self, t, fn):
        q = self._fired.get(t)
        self._at(q.pop(0) if q else t, fn)

    def kick(self):
        pass

    def run_to_completion(self):
        while self._q:
            self.now, _, fn = heapq.heappop(self._q)
            fn()
        return []

    def _emit(self, kind, h):
        ev = SimEvent(self.now, self._seq, kind, h.launch.task_id, h.launch.kernel_id, -1)
        self._seq += 1
        self.events.append(ev)
        if self.observer is not None:
            self.observer(ev)

    def submit(self, launch, at=None):
        sh = launch.shape
        got = (launch.task_id, launch.kernel_id, sh.kind,
               sh.worker_count if sh.kind == "ptb" else 0,
               sh.start_count if sh.kind == "ptb" else 0, launch.cost.total_blocks)
        self.submitted.append(got)
        if not self.expected:
            self.mismatch = self.mismatch or ("extra submission", got)
            rec = None
        else:
            rec = self.expected.popleft()
            tid, kid = self.names[(rec["task"], rec["kernel_index"])]
            want = (tid, kid, _SHAPES[rec["shape"]], rec["workers"] if rec["shape"] == 2 else 0,
                    rec["start_count"] if rec["shape"] == 2 else 0, rec["count"])
            if want != got and self.mismatch is None:
                self.mismatch = ("submission", len(self.submitted) - 1, want, got)
        h = _Handle(launch, rec)
        if rec is not None:
            self._at(max(self.now, rec["complete_ns"]), lambda: self._complete(h))
        return h

    def _complete(self, h):
        r = h.rec
        h.finish_time = self.now
        if r["parked"]:
            h.parked = True
            h.task_counter = r["task_counter"]
            self._emit(WORKER_PARKED, h)
        else:
            h.done = True
            h.task_counter = r["task_counter"]
            self._emit(KERNEL_FINISHED, h)

    def signal_preempt(self, h, at=None):
        if not h.is_ptb:
            raise ValueError(f"{h.launch.kernel_id}: not a Ptb launch")
        if h.done:
            raise ValueError(f"{h.launch.kernel_id}: not in flight")
        h.preempted = True
        self.preempts.append((h.launch.task_id, h.launch.kernel_id, h.shape.start_count))
        self._emit(PREEMPT_SIGNALED, h)


class FixedProfiler:
    """The B200 tuner's choices handed to the reference runner (its select is
    the only profiler call the runner makes, ref scheduler.py:372-376)."""

    def __init__(self, choices):
        self.choices = choices    # kernel_id -> ConfigCandidate

    def select(self, key, cost, threshold_ns=None):
        return self.choices[key.kernel]


def replay(gpu, tasks, config, horizon_ns, records, names, choices, timers=()):
    """Run the reference policy runner on ``ReplaySim``; returns the sim
    (``submitted``, ``preempts``, ``mismatch``) and the RunResult.
    ``timers``: the B200 run's (scheduled, fired) timer log."""
    from . import policy as pol
    sims = []

    def factory(g, placement_seed=0, record_events=True):
        s = ReplaySim(records, names, timers)
        sims.append(s)
        return s
    r = pol.PolicyRunner(gpu, tasks, config, horizon_ns, profiler=FixedProfiler(choices), sim_cls=factory)
    r.start_policy_clock()
    res = r.run()
    return sims[0], res


__all__ = ["ReplaySim", "FixedProfiler", "replay", "ConfigCandidate"]
