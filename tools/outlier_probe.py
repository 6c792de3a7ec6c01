"""Hunt the rare multi-millisecond HP stalls under co-location (C3 by
default): runs the solo and the co-located Tally window of one MMPP trace
several times with launch tracing and, for the requests whose co-located
latency exceeds their solo twin by more than --ms-threshold, prints the
request's own launch timeline (queue / issue / GPU start / GPU run / notice)
and the best-effort launches that were on the GPU in that interval.

    python tools/outlier_probe.py [--c2] [--ms 4000] [--reps 3] [--ms-threshold 1.5]
"""

from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import workloads  # noqa: E402


def arg(name, default):
    return type(default)(sys.argv[sys.argv.index(name) + 1]) if name in sys.argv else default


def main():
    from bench import c2_trace
    dev = P.B200Device.get(0)
    g = torch.Generator(device="cuda").manual_seed(0)
    if "--c2" in sys.argv:
        from paper_2410_07381_b200 import resnet
        hp = resnet.ResNet50Infer(batch=1, image=224)
        tr = resnet.ResNet50Train(batch=64, image=224, lr=0.01)
        tr.set_batch(torch.randn(64, 3, 224, 224, device="cuda", generator=g),
                     torch.randint(0, 1000, (64,), device="cuda", generator=g))
    else:
        from paper_2410_07381_b200 import gpt2
        hp = gpt2.BertInfer(seq=128)
        tr = gpt2.GPT2Train(batch=8, seq=1024, lr=1e-3)
        tr.set_batch(torch.randint(0, tr.V, (8, 1025), device="cuda", generator=g))
    prof = P.Profiler(dev.spec, runs=2)
    hp_w = P.KernelWork("hp", hp.kernel.cost(), exempt=True, kernel=hp.kernel)
    be_ws = []
    for name, dk in tr.program:
        sig = tr.work_signature(name, dk)
        prof.bind(sig, dk)
        be_ws.append(P.KernelWork(sig, dk.cost(), kernel=dk))
    lat = workloads.isolated_request_latency_ns(prof, (hp_w,))
    window = int(arg("--ms", 4000.0) * 1e6)
    thr = arg("--ms-threshold", 1.5) * 1e6
    cfg = P.SchedulerConfig(policy="Tally")
    out = []
    for rep in range(arg("--reps", 3)):
        arr = c2_trace(0.25, lat, window, arg("--seed", rep), 4.0)
        hp_t = P.TaskScript("hp", P.HIGH, (hp_w,), arr)
        be_t = P.TaskScript("be", P.BEST_EFFORT, tuple(be_ws))
        solo = P.run_policy(dev.spec, [hp_t], cfg, window, profiler=prof, record_events=False, options={"trace": 1})
        co = P.run_policy(dev.spec, [hp_t, be_t], cfg, window, profiler=prof, record_events=False,
                          options={"trace": 1})
        ds = dict(solo.requests["hp"])
        hp_l = [r for r in co.launches if r["priority"] == 0]
        be_l = [r for r in co.launches if r["priority"] != 0 and r["gpu_start_ns"] > 0]
        bad = []
        for (a, c), L in zip(co.requests["hp"], hp_l):
            if a in ds and (c - a) - (ds[a] - a) > thr:
                over = [dict(kind=be_ws[b["kernel_index"]].kernel_id.split(":")[0] if 0 <= b["kernel_index"] < len(be_ws) else "?",
                             shape=b["shape"], workers=b["workers"], start_us=round((b["gpu_start_ns"] - a) / 1e3),
                             run_us=round((b["gpu_end_ns"] - b["gpu_start_ns"]) / 1e3), parked=b["parked"])
                        for b in be_l if b["gpu_end_ns"] > a - 200_000 and b["gpu_start_ns"] < c]
                bad.append(dict(arrival_ms=round(a / 1e6, 2), solo_us=round((ds[a] - a) / 1e3), co_us=round((c - a) / 1e3),
                                queue_us=round((L["submit_ns"] - a) / 1e3), issue_us=round((L["issue_ns"] - L["submit_ns"]) / 1e3),
                                start_us=round((L["gpu_start_ns"] - L["issue_ns"]) / 1e3),
                                run_us=round((L["gpu_end_ns"] - L["gpu_start_ns"]) / 1e3),
                                notice_us=round((L["complete_ns"] - L["gpu_end_ns"]) / 1e3),
                                be_on_gpu=over[:12]))
        runs = [(round(L["gpu_start_ns"] / 1e6, 1), round((L["gpu_end_ns"] - L["gpu_start_ns"]) / 1e3))
                for L in hp_l if L["gpu_start_ns"] > 0]
        slow = [x for x in runs if x[1] > 2000]
        out.append({"rep": rep, "requests": len(co.requests["hp"]), "outliers": len(bad), "first": bad[:2],
                    "hp_graph_runs_over_2ms": len(slow), "slow_span_ms": [slow[0][0], slow[-1][0]] if slow else None,
                    "origin_ns": co.origin_ns})
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
