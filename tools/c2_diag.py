"""Config C2 co-location diagnostics: where does HP request latency go?

Runs one window of the C2 traffic (ResNet-50 bs=1 HP graph on the MMPP trace)
solo, and co-located with the ResNet-50 bs=64 training program under Tally
and KernelPriority, with GPU-timeline tracing.  For every HP request it
splits the latency into
  queue   arrival -> host submit (waiting for earlier requests)
  issue   host submit -> launch issued
  start   issue -> first GPU activity of the request's graph
  run     GPU start -> GPU end
  notice  GPU end -> completion observed by the daemon
and prints percentiles per policy, plus BE launch statistics.

    python tools/c2_diag.py [--ms 500] [--load 0.25] [--burst 4]
"""

from __future__ import annotations

import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import resnet, workloads  # noqa: E402


def arg(name, default):
    return type(default)(sys.argv[sys.argv.index(name) + 1]) if name in sys.argv else default


def pcts(xs):
    if not xs:
        return None
    s = sorted(xs)
    return [round(s[min(len(s) - 1, int(q * (len(s) - 1)))] / 1e3, 1) for q in (0.5, 0.9, 0.99)] + [round(s[-1] / 1e3, 1)]


def main():
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import ClockMap, c2_trace
    dev = P.B200Device.get(0)
    gpu = dev.spec
    window = int(arg("--ms", 500.0) * 1e6)
    load, burst = arg("--load", 0.25), arg("--burst", 4.0)
    threshold = int(arg("--threshold-us", 31.6) * 1000)
    g = torch.Generator(device="cuda").manual_seed(0)
    if "--c4" in sys.argv:
        from paper_2410_07381_b200 import bert, llama
        hp = llama.LlamaDecode(prompt=32, gen=arg("--gen", 16))
        tr = bert.BertTrain(batch=8, seq=512, lr=1e-3)
        tr.set_batch(torch.randint(0, tr.V, (8, 512), device="cuda", generator=g),
                     torch.randint(0, tr.V, (8, 512), device="cuda", generator=g))
    elif "--c3" in sys.argv:
        from paper_2410_07381_b200 import gpt2
        hp = gpt2.BertInfer(seq=128)
        tr = gpt2.GPT2Train(batch=8, seq=1024, lr=1e-3)
        tr.set_batch(torch.randint(0, tr.V, (8, 1025), device="cuda", generator=g))
    else:
        hp = resnet.ResNet50Infer(batch=1, image=224)
        tr = resnet.ResNet50Train(batch=64, image=224, lr=0.01)
        tr.set_batch(torch.randn(64, 3, 224, 224, device="cuda", generator=g),
                     torch.randint(0, 1000, (64,), device="cuda", generator=g))
    prof = P.Profiler(gpu, runs=2)
    if "--c4" in sys.argv:
        dec_w = P.KernelWork("decode_step", hp.decode_kernel.cost(), exempt=True, kernel=hp.decode_kernel)
        hp_pipe = (P.KernelWork("prefill", hp.prefill_kernel.cost(), exempt=True, kernel=hp.prefill_kernel),) + \
            (dec_w,) * hp.G
    else:
        hp_pipe = (P.KernelWork("hp_graph", hp.kernel.cost(), exempt=True, kernel=hp.kernel),)
    be_ws = []
    for name, dk in tr.program:
        sig = tr.work_signature(name, dk)
        prof.bind(sig, dk)
        be_ws.append(P.KernelWork(sig, dk.cost(), kernel=dk))
    hp_lat = workloads.isolated_request_latency_ns(prof, hp_pipe)
    chosen = [prof.select(w.profile_key(), w.cost, threshold) for w in be_ws]
    out = {"hp_isolated_us": hp_lat / 1e3,
           "choices": dict(collections.Counter(c.describe().split("(")[0] for c in chosen))}
    # chosen-config latency of the step vs untransformed
    lat_o = lat_c = 0
    worst = []
    for w, c in zip(be_ws, chosen):
        recs = prof.profile(w.profile_key(), w.cost)
        o = next(r for r in recs if r.candidate.variant == "Original")
        ch = next(r for r in recs if r.candidate == c)
        lat_o += o.kernel_latency_ns
        lat_c += ch.kernel_latency_ns
        worst.append((ch.kernel_latency_ns - o.kernel_latency_ns, w.kernel_id, c.describe(), o.kernel_latency_ns,
                      ch.kernel_latency_ns, ch.turnaround_estimate_ns))
    worst.sort(reverse=True)
    out["long_original_choices"] = sorted({(x[1], x[3], x[5]) for x in worst if x[2] == "Original" and x[3] > threshold},
                                          key=lambda t: -t[1])[:20]
    out["sliced_choices"] = sorted({(x[1], x[2], x[3], x[4], x[5]) for x in worst if x[2].startswith("Sliced")},
                                   key=lambda t: -t[3])[:20]
    out["profiled_step_ms"] = {"original": lat_o / 1e6, "chosen": lat_c / 1e6}
    out["worst_choices"] = [list(x) for x in worst[:12]]
    arr = c2_trace(load, hp_lat, window, 0, burst)
    hp_task = P.TaskScript("hp", P.HIGH, hp_pipe, arr)
    be_task = P.TaskScript("be", P.BEST_EFFORT, tuple(be_ws))
    for label, tasks, pol in (("be_solo", [be_task], "Tally"), ("solo", [hp_task], "Tally"),
                              ("tally", [hp_task, be_task], "Tally"),
                              ("kp", [hp_task, be_task], "KernelPriority")):
        cfg = P.SchedulerConfig(policy=pol, turnaround_threshold_ns=threshold)
        clk = ClockMap(dev)
        res = P.run_policy(gpu, tasks, cfg, window, profiler=prof, record_events=False, options={"trace": 1})
        clk.close()
        hp_l = [r for r in res.launches if r["priority"] == 0][::len(hp_pipe)]   # first step of each request
        be_l = [r for r in res.launches if r["priority"] != 0]
        reqs = res.requests.get("hp", [])
        q, iss, st, run, nt, tot = [], [], [], [], [], []
        for (a, c), L in zip(reqs, hp_l):
            q.append(L["submit_ns"] - a)
            iss.append(L["issue_ns"] - L["submit_ns"])
            if L["gpu_start_ns"] > 0:
                st.append(L["gpu_start_ns"] - L["issue_ns"])   # both run-relative
                run.append(L["gpu_end_ns"] - L["gpu_start_ns"])
                nt.append(L["complete_ns"] - L["gpu_end_ns"])
            tot.append(c - a)
        bykind = collections.defaultdict(list)
        for r in be_l:
            if r["preempt_ns"] < 0 or not r["parked"] or not r["gt_last_exit"]:
                continue
            sig = r["preempt_ns"] + res.origin_ns
            if r["gt_first_start"] and r["gt_first_start"] + clk.off(sig) >= sig:
                continue   # parked before any worker started (see bench.preempt_latencies_us)
            kind = be_ws[r["kernel_index"]].kernel_id.split(":")[0] if 0 <= r["kernel_index"] < len(be_ws) else "?"
            lat = ((r.get("gt_last_busy_exit") or r["gt_last_exit"]) + clk.off(sig) - sig) / 1e3
            drain = (r["gt_last_exit"] - r["gt_first_stop"]) / 1e3 if r["gt_first_stop"] else None
            bykind[kind].append((lat, drain, be_ws[r["kernel_index"]].kernel_id if 0 <= r["kernel_index"] < len(be_ws) else "?"))
        out[label + "_preempt_by_kind"] = {
            k: {"n": len(v), "lat_p50_max": [round(sorted(x[0] for x in v)[len(v) // 2], 1), round(max(x[0] for x in v), 1)],
                "drain_max": round(max((x[1] or 0) for x in v), 1),
                "worst": max(v)[2][:60]} for k, v in bykind.items()}
        out[label] = {"requests": len(reqs), "latency_p50_p90_p99_max_us": pcts(tot),
                      "queue": pcts(q), "issue": pcts(iss), "gpu_start": pcts(st), "gpu_run": pcts(run),
                      "notice": pcts(nt), "be_launches": len(be_l),
                      "be_iterations": len(res.iterations.get("be", ())),
                      "be_parked": sum(1 for r in be_l if r["parked"])}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
