"""Pin the CPU oracle (oracle/) against outputs of the reference itself.

Every expected value comes from tests/golden/*.json, written by
oracle/gen_golden.py running /root/reference's tallysim.  If these pass, the
oracle is a faithful restatement and may serve as the checker for the B200
path (and as the CPU baseline bench.py times).
"""

import hashlib
from fractions import Fraction

import pytest

from oracle import gpu_model as gm
from oracle import kernel_ir as ki
from oracle import policy as pol
from oracle import rewrites as rw
from oracle import traffic as tf
from oracle import tuner as tu


def _sha(s):
    return hashlib.sha256(s.encode()).hexdigest()


# ---------------------------------------------------------------- IR
def test_interpreter_matches_reference(gold):
    for case in gold("ir")["cases"]:
        k = ki.kernel_from_json(case["kernel"])
        r = ki.interpret(k, tuple(case["args"]), tuple(case["memory"]), case["seed"],
                         case["step_limit"])
        e = case["expect"]
        assert r.status == e["status"], case["name"]
        assert r.steps == e["steps"], case["name"]
        assert (None if r.memory is None else list(r.memory)) == e["memory"], case["name"]


def test_linearize_roundtrip_exhaustive():
    d = ki.Dim3(8, 8, 8)          # ref tests/test_ir.py:74-77
    for t in range(d.total):
        assert ki.linearize(ki.delinearize(t, d), d) == t
    assert ki.delinearize(13, ki.Dim3(4, 2, 3)) == ki.Dim3(1, 1, 1)


def test_wrap64():
    assert ki.wrap64(2 ** 63) == -2 ** 63
    assert ki.wrap64(-2 ** 63 - 1) == 2 ** 63 - 1
    assert ki.wrap64(5) == 5


def test_kernel_json_roundtrip(gold):
    for case in gold("ir")["cases"][:20]:
        k = ki.kernel_from_json(case["kernel"])
        assert ki.kernel_from_json(ki.kernel_to_json(k)) == k


# ---------------------------------------------------------------- transforms
def test_slice_extents_known_answers(gold):
    for e in gold("transforms")["extents"]:
        assert rw.slice_extents(e["len"], Fraction(e["frac"])) == e["extents"], e
    assert rw.slice_extents(10, Fraction(1, 4)) == [2] * 5      # half-even round
    with pytest.raises(rw.TransformError):
        rw.slice_extents(4, 0)


def test_slice_plans(gold):
    base = ki.kernel_from_json(gold("transforms")["equiv"][1]["kernel"])
    for p in gold("transforms")["plans"]:
        k = base.with_grid(ki.Dim3(*p["grid"]))
        plan = rw.slice_kernel(k, Fraction(p["frac"]))
        assert [[list(o), list(g)] for o, g in plan.subs] == p["subs"]


def test_sliced_and_ptb_equivalence(gold):
    for rec in gold("transforms")["equiv"]:
        k = ki.kernel_from_json(rec["kernel"])
        args, mem = tuple(rec["args"]), tuple(rec["memory"])
        base = ki.interpret(k, args, mem)
        assert list(base.memory) == rec["base"]["memory"]
        for f, exp in rec["sliced"].items():
            r = rw.run_sliced(rw.slice_kernel(k, Fraction(f)), args, mem)
            assert r.status == exp["status"]
            assert (r.memory == base.memory) == exp["same"]
            assert r.steps == exp["steps"]
        for w, exp in rec["ptb"].items():
            wk = rw.make_preemptible(rw.unify_synchronization(k), ki.Dim3(int(w)))
            n = len(mem)
            ctl = rw.PtbControl(n, n + 1, k.grid.total, k.grid)
            r = rw.run_ptb(wk, ctl, args, mem + (0, 0))
            assert r.status == exp["status"]
            assert list(r.memory[n:]) == exp["tail"]
            assert (r.memory[:n] == base.memory) == exp["same"]


def test_preempt_resume_every_counter(gold):
    g = gold("transforms")["preempt"]
    k = ki.kernel_from_json(g["kernel"])
    wk = rw.make_preemptible(rw.unify_synchronization(k), ki.Dim3(g["workers"]))
    ctl = rw.PtbControl(g["ctr"], g["flag"], 16, k.grid)
    args, mem = tuple(g["args"]), tuple(g["memory"])
    assert list(rw.run_ptb(wk, ctl, args, mem).memory) == g["uninterrupted"]["memory"]
    for s in g["sweep"]:
        first = rw.run_ptb(wk, ctl, args, mem, preempt_at_count=s["c"])
        assert list(first.memory) == s["first"]["memory"]
        m = list(first.memory)
        m[g["flag"]] = 0
        second = rw.run_ptb(wk, ctl, args, tuple(m))
        assert list(second.memory) == s["second"]["memory"]


def test_unified_sync_witness(gold):
    w = gold("transforms")["witness"]
    k = ki.kernel_from_json(w["kernel"])
    raw = rw.run_ptb(rw.make_preemptible(k, ki.Dim3(1), enforce_unified=False),
                     rw.PtbControl(4, 5, 4, k.grid), (), (0,) * 6)
    assert raw.status == w["raw"]["status"] == ki.DIVERGENT_BARRIER
    uni = rw.run_ptb(rw.make_preemptible(rw.unify_synchronization(k), ki.Dim3(1)),
                     rw.PtbControl(4, 5, 2, k.grid), (), (0,) * 6)
    assert list(uni.memory) == w["unified"]["memory"]
    assert list(uni.memory[:4]) == [7, 7, 7, 7]


# ---------------------------------------------------------------- sim
def _shape(d):
    if d["kind"] == "sliced":
        return gm.SlicedShape(tuple(d["sub_blocks"]))
    if d["kind"] == "ptb":
        return gm.PtbShape(d["worker_count"], d["start_count"])
    return gm.OriginalShape()


def _cost(d):
    return gm.KernelCostModel(**d)


def test_sim_event_logs_byte_identical(gold):
    for sc in gold("sim")["scenarios"]:
        s = gm.GpuSim(gm.GpuSpec(*sc["gpu"]), placement_seed=sc["seed"])
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


# ---------------------------------------------------------------- tuner
def _cand(d):
    return tu.ConfigCandidate(d["variant"], Fraction(d["fraction"]) if d["fraction"] else None,
                              d["worker_count"])


def test_candidate_menus(gold):
    for m in gold("tuner")["menus"]:
        got = tu.candidate_configs(gm.cost_model(0.1, m["blocks"], m["tpb"]), gm.GpuSpec(*m["gpu"]))
        assert got == [_cand(c) for c in m["cands"]], m


def test_eq1_known_answers(gold):
    for e in gold("tuner")["eq1"]:
        c = tu.ConfigCandidate("Ptb", worker_count=e["w"])
        assert tu.estimate_turnaround(c, e["lat"], e["total"]) == e["est"]


def test_profiles_and_selection(gold):
    for p in gold("tuner")["profiles"]:
        prof = tu.Profiler(gm.GpuSpec(*p["gpu"]), runs=p["runs"])
        for name, ms, blocks, tpb in p["items"]:
            key = tu.ProfileKey(name, (blocks, 1, 1), (tpb, 1, 1))
            recs = prof.profile(key, gm.cost_model(ms, blocks, tpb))
            for th, c in p["select"][name].items():
                assert tu.select_config(recs, int(th)) == _cand(c), (name, th)
        assert prof.dump_cache() == p["cache"]
        assert prof.simulated_runs == p["simulated_runs"]
        again = tu.Profiler(gm.GpuSpec(*p["gpu"]))
        again.load_cache(p["cache"])
        assert again.dump_cache() == p["cache"]


# ---------------------------------------------------------------- policy
def _scenarios():
    KW, TS = pol.KernelWork, pol.TaskScript
    cm, ms = gm.cost_model, gm.ms_to_ns
    HIGH, BE = gm.HIGH, gm.BEST_EFFORT
    G4, GB = gm.GpuSpec(4, 128, 1), gm.GpuSpec(148, 2048, 32)
    hp, be = cm(1.0, 1, threads_per_block=128), cm(0.15, 108, threads_per_block=128)
    arr = tuple(ms(x) for x in (0.5, 3.0, 3.2, 7.7, 12.0, 12.0, 15.3))
    varr = tuple(ms(x) for x in (0.01, 0.07, 0.08, 0.2, 0.33, 0.34, 0.5, 0.71))
    return {
        "hp_be": (G4, 20.0, [TS("hp", HIGH, (KW("hp_k", hp),), arr), TS("be", BE, (KW("be_k", be),))]),
        "two_be": (G4, 10.0, [TS("hp", HIGH, (KW("hp_k", hp),), arr[:3]),
                              TS("b1", BE, (KW("b1_k", be),)),
                              TS("b2", BE, (KW("b2_k", cm(0.4, 16, 128)),))]),
        "exempt": (G4, 8.0, [TS("hp", HIGH, (KW("hp_k", hp),), arr[:3]),
                             TS("be", BE, (KW("be_k", be, exempt=True),))]),
        "pipeline": (G4, 12.0, [TS("hp", HIGH, (KW("h1", cm(0.3, 2, 128)), KW("h2", cm(0.2, 6, 128))), arr[:5]),
                                TS("be", BE, (KW("e1", cm(0.05, 40, 128)), KW("e2", cm(0.4, 9, 128)),
                                              KW("e3", cm(2.0, 3, 128))))]),
        "sliced_be": (G4, 6.0, [TS("hp", HIGH, (KW("hp_k", cm(0.2, 1, 128)),), (ms(1.1), ms(2.9))),
                                TS("be", BE, (KW("be_k", cm(0.5, 16, 128)),))]),
        "be_inference": (G4, 10.0, [TS("hp", HIGH, (KW("hp_k", hp),), arr[:4]),
                                    TS("bi", BE, (KW("bi_k", cm(0.3, 8, 128)),),
                                       tuple(ms(x) for x in (0.1, 0.2, 2.0, 2.05, 6.0)))]),
        "b200_c1": (GB, 1.0, [TS("hp", HIGH, (KW("vadd", cm(0.004, 4096, 256)),), varr),
                              TS("be", BE, (KW("sgemm", cm(0.03, 2048, 256)),))]),
    }


POLICY_SCENARIOS = _scenarios


@pytest.mark.parametrize("name", list(_scenarios()))
def test_policy_runs_match_reference(gold, name):
    gpu, hz, tasks = _scenarios()[name]
    runs = [r for r in gold("policy")["runs"] if r["scenario"] == name]
    prof = tu.Profiler(gpu, runs=runs[0]["runs"])
    for r in runs:
        cfg = pol.SchedulerConfig(policy=r["policy"], **(
            {"turnaround_threshold_ns": r["threshold"]} if "threshold" in r else {}))
        res = pol.run_policy(gpu, tasks, cfg, gm.ms_to_ns(hz), profiler=prof,
                             placement_seed=r["seed"])
        assert _sha(gm.events_to_csv(res.events)) == r["csv_sha256"], (name, r["policy"])
        assert {k: [list(x) for x in v] for k, v in res.requests.items()} == r["requests"]
        assert res.iterations == r["iterations"]


# ---------------------------------------------------------------- traffic
def test_arrivals_and_p99(gold):
    g = gold("traffic")
    for a in g["arrivals"]:
        got = tf.generate_arrivals(a["load"], a["lat"], a["dur"], a["seed"])
        assert len(got) == a["n"] and list(got[:20]) == a["head"]
        assert _sha(",".join(map(str, got))) == a["sha256"]
    for p in g["p99"]:
        assert tf.p99_nearest_rank(p["xs"]) == p["p99"]


def test_desk_experiment_rows(gold):
    g = gold("traffic")["experiment"]
    KW = pol.KernelWork
    serve = tf.WorkloadSpec("serve", "inference", gm.HIGH,
                            (KW("serve_k", gm.cost_model(3.925, 1, threads_per_block=128)),),
                            tf.TraceSpec(load=0.5))
    train = tf.WorkloadSpec("train", "training", gm.BEST_EFFORT,
                            (KW("train_k", gm.cost_model(0.15, 108, threads_per_block=128)),))
    reps = tf.run_experiment(gm.GpuSpec(4, 128, 1), [serve, train],
                             ["Tally", "KernelPriority", "Eager", "TimeSliced"],
                             gm.ms_to_ns(g["horizon_ms"]), seed=0)
    assert [row for r in reps for row in tf.report_csv_rows(r)] == g["rows"]
