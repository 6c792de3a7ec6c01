"""Where does the runtime's per-kernel gap go?  Runs the C2 training program
alone through run_policy (Eager: every kernel untransformed, one in flight)
with GPU-timeline tracing and splits the time between consecutive BE kernels:

  notice  GPU end of kernel k   -> daemon observes completion
  decide  completion observed   -> kernel k+1 submitted (runner tick)
  issue   submit                -> launch API returned
  start   launch issued         -> GPU start of kernel k+1

    python tools/runner_gaps.py [--policy Eager|Tally]
"""

from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import resnet  # noqa: E402


def pcts(xs):
    s = sorted(xs)
    return [round(s[int(q * (len(s) - 1))] / 1e3, 2) for q in (0.1, 0.5, 0.9, 0.99)] + [round(sum(s) / 1e6, 2)]


def main():
    pol = sys.argv[sys.argv.index("--policy") + 1] if "--policy" in sys.argv else "Eager"
    dev = P.B200Device.get(0)
    tr = resnet.ResNet50Train(batch=64, image=224, lr=0.01)
    g = torch.Generator(device="cuda").manual_seed(0)
    tr.set_batch(torch.randn(64, 3, 224, 224, device="cuda", generator=g),
                 torch.randint(0, 1000, (64,), device="cuda", generator=g))
    prof = P.Profiler(dev.spec, runs=1)
    works = []
    for name, dk in tr.program:
        sig = tr.work_signature(name, dk)
        prof.bind(sig, dk)
        works.append(P.KernelWork(sig, dk.cost(), kernel=dk))
    be = P.TaskScript("be", P.BEST_EFFORT, tuple(works))
    cfg = P.SchedulerConfig(policy=pol)
    P.run_policy(dev.spec, [be], cfg, int(100e6), profiler=prof, record_events=False)   # warm + profile
    res = P.run_policy(dev.spec, [be], cfg, int(300e6), profiler=prof, record_events=False, options={"trace": 1})
    L = sorted((r for r in res.launches if r["gpu_start_ns"] > 0), key=lambda r: r["submit_ns"])
    notice, decide, issue, start, run = [], [], [], [], []
    for a, b in zip(L, L[1:]):
        notice.append(a["complete_ns"] - a["gpu_end_ns"])
        decide.append(b["submit_ns"] - a["complete_ns"])
        issue.append(b["issue_ns"] - b["submit_ns"])
        start.append(b["gpu_start_ns"] - b["issue_ns"])
        run.append(a["gpu_end_ns"] - a["gpu_start_ns"])
    it = res.iterations["be"]
    print(json.dumps({"policy": pol, "launches": len(L), "iterations": len(it),
                      "step_ms": (it[-1] - it[0]) / 1e6 / max(1, len(it) - 1) if len(it) > 1 else None,
                      "p10_p50_p90_p99_us_total_ms": {"notice": pcts(notice), "decide": pcts(decide),
                                                      "issue": pcts(issue), "start": pcts(start),
                                                      "gpu_run": pcts(run)}}, indent=1))


if __name__ == "__main__":
    main()
