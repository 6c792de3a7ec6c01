"""Co-location diagnostics on the B200: HP vecadd at Poisson arrivals next to a
BE kernel loop under each policy; prints the tuner's choice, HP latency
percentiles, BE iterations and per-launch preemption telemetry as JSON.

    python tools/colo_diag.py [--be vecadd_f32|rowsum_f32|sgemm_tf32x3|gemm_bf16] [--ms 200]
"""

from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import kernels, workloads  # noqa: E402


def arg(name, default):
    return type(default)(sys.argv[sys.argv.index(name) + 1]) if name in sys.argv else default


def _pick(recs, f, q):
    xs = sorted(f(r) for r in recs if r["priority"] == 0 and r["gpu_start_ns"] >= 0)
    return xs[min(len(xs) - 1, int(q * (len(xs) - 1)))] / 1e3 if xs else None


def _q(recs, q):   # issue -> GPU start (queueing for SM resources / stream)
    return _pick(recs, lambda r: r["gpu_start_ns"] - r["issue_ns"], q)


def _r(recs, q):   # GPU start -> end
    return _pick(recs, lambda r: r["gpu_end_ns"] - r["gpu_start_ns"], q)


def _h(recs, q):   # host submit -> issue
    return _pick(recs, lambda r: r["issue_ns"] - r["submit_ns"], q)


def main():
    dev = P.B200Device.get(0)
    be_kind = arg("--be", "vecadd_f32")
    horizon = int(arg("--ms", 200.0) * 1e6)
    load = arg("--load", 0.5)
    threshold = int(arg("--threshold-us", 31.6) * 1000)
    if "--host-flag" in sys.argv:
        dev.set_flag_mode(True)
    g = torch.Generator(device="cuda").manual_seed(0)
    n = 1 << 24
    a, b, c = (torch.rand(n, device="cuda", generator=g) for _ in range(3))
    hp = kernels.vecadd_f32(a, b, c)
    if be_kind == "vecadd_f32":
        bufs = [torch.rand(1 << 26, device="cuda", generator=g) for _ in range(3)]
        be = kernels.vecadd_f32(*bufs)
    elif be_kind == "rowsum_f32":
        x = torch.rand(1 << 16, 1024, device="cuda", generator=g)
        be = kernels.rowsum_f32(x, torch.zeros(1 << 16, device="cuda"))
    elif be_kind == "sgemm_pipeline":
        A = torch.rand(4096, 4096, device="cuda", generator=g) * 2 - 1
        B = torch.rand(4096, 4096, device="cuda", generator=g) * 2 - 1
        sg = kernels.sgemm_tf32x3(A, B, torch.zeros(4096, 4096, device="cuda"))
        be = sg.gemm
    else:
        from tools.microbench import make
        be = make(be_kind)
    prof = P.Profiler(dev.spec, runs=5)
    hp_w = P.KernelWork("vadd_hp", hp.cost(), kernel=hp)
    be_w = P.KernelWork(be_kind, be.cost(), kernel=be)
    prof.bind("vadd_hp", hp)
    prof.bind(be_kind, be)
    be_ws = (be_w,)
    if be_kind == "sgemm_pipeline":
        be_ws = (P.KernelWork("split_a", sg.split_a.cost(), kernel=sg.split_a),
                 P.KernelWork("split_b", sg.split_b.cost(), kernel=sg.split_b), be_w)
        for w in be_ws:
            prof.bind(w.kernel_id, w.kernel)
    hp_lat = workloads.isolated_request_latency_ns(prof, (hp_w,))
    arr = workloads.generate_arrivals(load, hp_lat, horizon, seed=0)
    recs = prof.profile(be_w.profile_key(), be_w.cost)
    out = {"hp_isolated_latency_us": hp_lat / 1e3, "arrivals": len(arr),
           "be_profile": [(r.candidate.describe(), r.kernel_latency_ns / 1e3,
                           r.turnaround_estimate_ns / 1e3) for r in recs],
           "be_choice": prof.select(be_w.profile_key(), be_w.cost, threshold).describe(),
           "policies": {}}
    off, _ = dev.clock_offset()
    for pol in ("Tally", "KernelPriority", "Eager"):
        cfg = P.SchedulerConfig(policy=pol, turnaround_threshold_ns=threshold)
        hp_t = P.TaskScript("hp", P.HIGH, (hp_w,), arr)
        be_t = P.TaskScript("be", P.BEST_EFFORT, be_ws)
        solo_hp = P.run_policy(dev.spec, [hp_t], cfg, horizon, profiler=prof, record_events=False,
                               options={"trace": 1})
        solo_be = P.run_policy(dev.spec, [be_t], cfg, horizon, profiler=prof, record_events=False)
        co = P.run_policy(dev.spec, [hp_t, be_t], cfg, horizon, profiler=prof, record_events=False,
                          options={"trace": 1})
        # the five slowest HP requests: host submit/issue/complete vs GPU start/end
        hp_l = sorted((r for r in co.launches if r["priority"] == 0),
                      key=lambda r: r["complete_ns"] - r["submit_ns"])[-5:]
        worst = []
        for r in hp_l:
            near = [(b["shape"], b["issue_ns"] / 1e3, b["gpu_start_ns"] / 1e3, b["gpu_end_ns"] / 1e3,
                     b["complete_ns"] / 1e3, b["parked"])
                    for b in co.launches if b["priority"] == 1 and
                    b["gpu_end_ns"] >= r["submit_ns"] - 50_000 and b["issue_ns"] <= r["complete_ns"]]
            worst.append({"submit": r["submit_ns"] / 1e3, "issue": r["issue_ns"] / 1e3,
                          "gpu_start": r["gpu_start_ns"] / 1e3, "gpu_end": r["gpu_end_ns"] / 1e3,
                          "complete": r["complete_ns"] / 1e3, "be_near": near[:6]})
        m_solo = workloads.compute_task_metrics(solo_hp)["hp"]
        m_co = workloads.compute_task_metrics(co)
        be_solo = workloads.compute_task_metrics(solo_be)["be"]
        lat = sorted(c - a for a, c in co.requests["hp"])
        slat = sorted(c - a for a, c in solo_hp.requests["hp"])
        pre = [r for r in co.launches if r["preempt_ns"] >= 0 and r["parked"]]
        pl = sorted((r["gt_last_exit"] + off - (r["preempt_ns"] + co.origin_ns)) / 1e3 for r in pre)
        out["policies"][pol] = {
            "hp_p50_us": [slat[len(slat) // 2] / 1e3, lat[len(lat) // 2] / 1e3],
            "hp_p99_us": [m_solo.p99_latency_ns / 1e3, m_co["hp"].p99_latency_ns / 1e3],
            "hp_max_us": [slat[-1] / 1e3, lat[-1] / 1e3],
            "p99_overhead_pct": 100 * (m_co["hp"].p99_latency_ns / m_solo.p99_latency_ns - 1),
            "be_iters_per_s": [be_solo.throughput_per_s, m_co["be"].throughput_per_s],
            "be_fraction": m_co["be"].throughput_per_s / be_solo.throughput_per_s,
            "be_launches": sum(1 for r in co.launches if r["priority"] == 1),
            "preempts": len(pre),
            "preempt_us_p50_p99_max": [pl[len(pl) // 2], pl[int(0.99 * (len(pl) - 1))], pl[-1]] if pl else None,
            "worst_hp": worst,
            "hp_queue_us_p50_p99_solo_co": [
                _q(solo_hp.launches, 0.5), _q(solo_hp.launches, 0.99), _q(co.launches, 0.5), _q(co.launches, 0.99)],
            "hp_run_us_p50_p99_solo_co": [
                _r(solo_hp.launches, 0.5), _r(solo_hp.launches, 0.99), _r(co.launches, 0.5), _r(co.launches, 0.99)],
            "hp_host_issue_us_p50_p99_solo_co": [
                _h(solo_hp.launches, 0.5), _h(solo_hp.launches, 0.99), _h(co.launches, 0.5), _h(co.launches, 0.99)],
        }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
