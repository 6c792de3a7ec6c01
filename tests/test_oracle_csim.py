"""Pin the C restatement of the reference GPU (oracle/csim.c) to the reference.

The same golden vectors as tests/test_oracle_golden.py (written by running
/root/reference's tallysim): simulator event logs byte-identical, tuner
records and cache JSON identical, and every policy run's event log identical
when the policy runner and the profiler drive the C simulator.  bench.py's CPU
reference arm runs on this simulator, so these tests are what make its
numbers the reference algorithm's.
"""

import hashlib
import random

import pytest

from oracle import csim
from oracle import gpu_model as gm
from oracle import policy as pol
from oracle import tuner as tu
from test_oracle_golden import _cand, _cost, _scenarios, _shape


def _sha(s):
    return hashlib.sha256(s.encode()).hexdigest()


def test_csim_event_logs_byte_identical(gold):
    for sc in gold("sim")["scenarios"]:
        s = csim.GpuSim(gm.GpuSpec(*sc["gpu"]), placement_seed=sc["seed"])
        hs = [s.submit(gm.SimLaunch(l["task"], l["kernel"], l["priority"], _shape(l["shape"]),
                                    _cost(l["cost"])), l["at"]) for l in sc["launches"]]
        for p in sc["preempts"]:
            s.signal_preempt(hs[p["launch"]], p["at"])
        s.run_to_completion()
        csv = gm.events_to_csv(s.events)
        if sc["csv"] is not None:
            assert csv == sc["csv"], sc["name"]
        assert _sha(csv) == sc["csv_sha256"], sc["name"]
        for h, e in zip(hs, sc["handles"]):
            assert h.finish_time == e["finish_time"], sc["name"]
            assert h.blocks_finished == e["blocks_finished"]
            assert h.task_counter == e["task_counter"]
            assert h.park_times == e["park_times"]
            assert h.sub_completions == e["sub_completions"]
        for p, t in zip(sc["preempts"], sc["turnaround"]):
            if t is not None:
                assert s.measured_turnaround(hs[p["launch"]], p["at"]) == t


def test_csim_profiles_and_selection(gold):
    for p in gold("tuner")["profiles"]:
        prof = tu.Profiler(gm.GpuSpec(*p["gpu"]), runs=p["runs"], sim_cls=csim.GpuSim)
        for name, ms, blocks, tpb in p["items"]:
            key = tu.ProfileKey(name, (blocks, 1, 1), (tpb, 1, 1))
            recs = prof.profile(key, gm.cost_model(ms, blocks, tpb))
            for th, c in p["select"][name].items():
                assert tu.select_config(recs, int(th)) == _cand(c), (name, th)
        assert prof.dump_cache() == p["cache"]


@pytest.mark.parametrize("name", list(_scenarios()))
def test_csim_policy_runs_match_reference(gold, name):
    gpu, hz, tasks = _scenarios()[name]
    runs = [r for r in gold("policy")["runs"] if r["scenario"] == name]
    prof = tu.Profiler(gpu, runs=runs[0]["runs"], sim_cls=csim.GpuSim)
    for r in runs:
        cfg = pol.SchedulerConfig(policy=r["policy"], **(
            {"turnaround_threshold_ns": r["threshold"]} if "threshold" in r else {}))
        res = pol.run_policy(gpu, tasks, cfg, gm.ms_to_ns(hz), profiler=prof,
                             placement_seed=r["seed"], sim_cls=csim.GpuSim)
        assert _sha(gm.events_to_csv(res.events)) == r["csv_sha256"], (name, r["policy"])
        assert {k: [list(x) for x in v] for k, v in res.requests.items()} == r["requests"]
        assert res.iterations == r["iterations"]


def test_csim_matches_python_oracle_on_random_preemptions():
    """Random mixes of all three shapes with random preempt times: identical
    event logs and handle states from the Python and the C event loop."""
    for seed in range(12):
        rng = random.Random(seed)
        gpu = gm.GpuSpec(rng.choice((4, 16, 148)), rng.choice((256, 2048)), rng.choice((1, 8, 32)))
        sims = [gm.GpuSim(gpu, placement_seed=seed), csim.GpuSim(gpu, placement_seed=seed)]
        plans = []
        for i in range(rng.randint(2, 7)):
            total = rng.randint(1, 300)
            tpb = rng.choice((32, 128, 256))
            cost = gm.KernelCostModel(rng.randint(1, 5000), rng.randint(0, 3000), rng.randint(0, 300), tpb, total)
            kind = rng.choice(("original", "sliced", "ptb"))
            if kind == "sliced" and total > 1:
                k = rng.randint(2, min(total, 6))
                cuts = sorted(rng.sample(range(1, total), k - 1))
                shape = gm.SlicedShape(tuple(b - a for a, b in zip([0] + cuts, cuts + [total])))
            elif kind == "ptb":
                shape = gm.PtbShape(rng.randint(1, 64), rng.randint(0, total - 1))
            else:
                shape = gm.OriginalShape()
            prio = rng.choice((gm.HIGH, gm.BEST_EFFORT))
            plans.append((gm.SimLaunch(f"t{i}", f"k{i}", prio, shape, cost), rng.randint(0, 20000)))
        pre = [(i, rng.randint(0, 40000)) for i, (l, _) in enumerate(plans) if l.shape.kind == "ptb"
               and rng.random() < 0.7]
        logs = []
        for s in sims:
            hs = [s.submit(l, at) for l, at in plans]
            for i, t in pre:
                s.signal_preempt(hs[i], t)
            s.run_to_completion()
            logs.append((gm.events_to_csv(s.events),
                         [(h.finish_time, h.blocks_finished, h.task_counter, h.park_times, h.sub_completions,
                           h.parked, h.done) for h in hs], s._nlogged))
        assert logs[0] == logs[1], seed
