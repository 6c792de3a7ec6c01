"""The product's decision core against the reference (CPU, no GPU needed).

* The native policy runner (libtally_b200 ``tally_runner_*``) drives the CPU
  oracle's virtual-time GPU through the ``tally_device_vtbl`` callbacks; its
  event log must equal the reference's byte for byte, for every policy,
  scenario, placement seed and threshold in tests/golden/policy.json.
* The product profiler, measuring on the injected virtual device, must
  reproduce the reference's profile records, cache JSON and selections.
* Pure tuner/tiling arithmetic must match the reference's known answers.
"""

import hashlib
from fractions import Fraction

import pytest

import paper_2410_07381_b200 as P
from paper_2410_07381_b200 import profiler as pp
from paper_2410_07381_b200 import transforms as pt
from paper_2410_07381_b200 import workloads as pw
from oracle import gpu_model as gm
from test_oracle_golden import _scenarios


def _sha(s):
    return hashlib.sha256(s.encode()).hexdigest()


def _product_tasks(tasks):
    return [P.TaskScript(t.task_id, t.priority,
                         tuple(P.KernelWork(w.kernel_id, w.cost, w.exempt) for w in t.kernels),
                         t.arrivals) for t in tasks]


@pytest.mark.parametrize("name", list(_scenarios()))
def test_native_runner_event_log_matches_reference(gold, name):
    gpu, hz, tasks = _scenarios()[name]
    runs = [r for r in gold("policy")["runs"] if r["scenario"] == name]
    prof = P.Profiler(gpu, runs=runs[0]["runs"], device_factory=gm.GpuSim)
    ptasks = _product_tasks(tasks)
    for r in runs:
        kw = {"turnaround_threshold_ns": r["threshold"]} if "threshold" in r else {}
        res = P.run_policy(gpu, ptasks, P.SchedulerConfig(policy=r["policy"], **kw),
                           P.ms_to_ns(hz), profiler=prof, placement_seed=r["seed"],
                           device_factory=gm.GpuSim)
        assert _sha(P.events_to_csv(res.events)) == r["csv_sha256"], (name, r["policy"], r["seed"])
        assert {k: [list(x) for x in v] for k, v in res.requests.items()} == r["requests"]
        assert res.iterations == r["iterations"]


def _cand(d):
    return pp.ConfigCandidate(d["variant"], Fraction(d["fraction"]) if d["fraction"] else None,
                              d["worker_count"])


def test_candidate_menus(gold):
    for m in gold("tuner")["menus"]:
        got = pp.candidate_configs(P.cost_model(0.1, m["blocks"], m["tpb"]), P.GpuSpec(*m["gpu"]))
        assert got == [_cand(c) for c in m["cands"]], m


def test_eq1(gold):
    for e in gold("tuner")["eq1"]:
        c = pp.ConfigCandidate("Ptb", worker_count=e["w"])
        assert pp.estimate_turnaround(c, e["lat"], e["total"]) == e["est"]


def test_profiler_records_and_selection(gold):
    for p in gold("tuner")["profiles"]:
        prof = P.Profiler(P.GpuSpec(*p["gpu"]), runs=p["runs"], device_factory=gm.GpuSim)
        for name, ms, blocks, tpb in p["items"]:
            key = P.ProfileKey(name, (blocks, 1, 1), (tpb, 1, 1))
            recs = prof.profile(key, P.cost_model(ms, blocks, tpb))
            for th, c in p["select"][name].items():
                assert P.select_config(recs, int(th)) == _cand(c), (name, th)
        assert prof.dump_cache() == p["cache"]
        assert prof.simulated_runs == p["simulated_runs"]
        again = P.Profiler(P.GpuSpec(*p["gpu"]))
        again.load_cache(p["cache"])
        assert again.dump_cache() == p["cache"]


def test_slice_extents_and_plans(gold):
    g = gold("transforms")
    for e in g["extents"]:
        assert pt.slice_extents(e["len"], Fraction(e["frac"])) == e["extents"]
    for p in g["plans"]:
        plan = pt.slice_plan(None, Fraction(p["frac"]), grid=p["grid"])
        assert [[list(o), list(s)] for o, s in plan] == p["subs"]
    # linear plan covers every logical block exactly once
    for total in (1, 7, 100, 2048):
        for f in (Fraction(1, 2), Fraction(1, 3), Fraction(1, total)):
            cover = [i for off, n in pt.slice_plan(total, f) for i in range(off, off + n)]
            assert cover == list(range(total))
    with pytest.raises(P.TransformError):
        pt.slice_extents(4, Fraction(3, 2))


def test_linearize_roundtrip():
    d = (8, 8, 8)
    for t in range(512):
        assert pt.linearize(pt.delinearize(t, d), d) == t


def test_runner_errors_map_to_reference_exceptions():
    gpu = P.GpuSpec(4, 128, 1)
    with pytest.raises(ValueError):
        P.SchedulerConfig(policy="Fifo")
    with pytest.raises(ValueError):
        P.TaskScript("t", P.HIGH, ())
    w = P.KernelWork("k", P.cost_model(0.1, 4, 128))
    with pytest.raises(ValueError):
        P.run_policy(gpu, [P.TaskScript("x", P.BEST_EFFORT, (w,)),
                           P.TaskScript("x", P.BEST_EFFORT, (w,))],
                     P.SchedulerConfig(), 1_000_000, device_factory=gm.GpuSim)
    # a B200 run without a bound device kernel is refused loudly
    with pytest.raises(ValueError):
        P.run_policy(gpu, [P.TaskScript("x", P.HIGH, (w,), (10,))],
                     P.SchedulerConfig(policy="Eager"), 1_000_000)


def test_desk_experiment_rows_through_native_runner(gold):
    g = gold("traffic")["experiment"]
    serve = pw.WorkloadSpec("serve", "inference", P.HIGH,
                            (P.KernelWork("serve_k", P.cost_model(3.925, 1, threads_per_block=128)),),
                            pw.TraceSpec(load=0.5))
    train = pw.WorkloadSpec("train", "training", P.BEST_EFFORT,
                            (P.KernelWork("train_k", P.cost_model(0.15, 108, threads_per_block=128)),))
    reps = pw.run_experiment(P.GpuSpec(4, 128, 1), [serve, train],
                             ["Tally", "KernelPriority", "Eager", "TimeSliced"],
                             P.ms_to_ns(g["horizon_ms"]), seed=0, device_factory=gm.GpuSim)
    assert [row for r in reps for row in pw.report_csv_rows(r)] == g["rows"]


def test_arrivals_match_reference(gold):
    for a in gold("traffic")["arrivals"]:
        got = pw.generate_arrivals(a["load"], a["lat"], a["dur"], a["seed"])
        assert _sha(",".join(map(str, got))) == a["sha256"]
    for p in gold("traffic")["p99"]:
        assert pw.p99_nearest_rank(p["xs"]) == p["p99"]


def test_bursty_trace_roundtrip(tmp_path):
    path = tmp_path / "burst.csv"
    n = pw.bursty_trace(str(path), mean_gap_ms=1.0, duration_ms=2000.0, seed=3)
    stamps = pw.load_trace(str(path))
    assert len(stamps) == n > 100
    assert all(b >= a for a, b in zip(stamps, stamps[1:]))
    gaps = [b - a for a, b in zip(stamps, stamps[1:])]
    # bursty: coefficient of variation well above Poisson's 1
    mean = sum(gaps) / len(gaps)
    cv = (sum((x - mean) ** 2 for x in gaps) / len(gaps)) ** 0.5 / mean
    assert cv > 1.5
