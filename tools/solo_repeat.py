"""Is the solo high-priority p99 reproducible?  Runs the same MMPP arrival
trace through the runner (HP alone, Tally policy) several times and prints
each run's p50 / p99 / max request latency and the largest per-request
difference between runs.

    python tools/solo_repeat.py [--c2] [--ms 4000] [--reps 4]
"""

from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import workloads  # noqa: E402


def arg(name, default):
    return type(default)(sys.argv[sys.argv.index(name) + 1]) if name in sys.argv else default


def main():
    from bench import c2_trace, p99
    dev = P.B200Device.get(0)
    if "--c2" in sys.argv:
        from paper_2410_07381_b200 import resnet
        hp = resnet.ResNet50Infer(batch=1, image=224)
    else:
        from paper_2410_07381_b200 import gpt2
        hp = gpt2.BertInfer(seq=128)
    prof = P.Profiler(dev.spec, runs=2)
    w = P.KernelWork("hp", hp.kernel.cost(), exempt=True, kernel=hp.kernel)
    lat = workloads.isolated_request_latency_ns(prof, (w,))
    window = int(arg("--ms", 4000.0) * 1e6)
    arr = c2_trace(0.25, lat, window, 1, 4.0)
    task = P.TaskScript("hp", P.HIGH, (w,), arr)
    cfg = P.SchedulerConfig(policy="Tally")
    runs = []
    for _ in range(arg("--reps", 4)):
        r = P.run_policy(dev.spec, [task], cfg, window, profiler=prof, record_events=False)
        runs.append(dict(r.requests["hp"]))
    out = []
    for d in runs:
        ls = sorted(c - a for a, c in d.items())
        out.append({"n": len(ls), "p50_us": ls[len(ls) // 2] / 1e3, "p99_us": p99(ls) / 1e3, "max_us": ls[-1] / 1e3})
    diffs = [abs((runs[i][a] - a) - (runs[0][a] - a)) / 1e3 for i in range(1, len(runs)) for a in runs[0] if a in runs[i]]
    print(json.dumps({"isolated_us": lat / 1e3, "runs": out, "max_request_diff_us": max(diffs) if diffs else None,
                      "p99_request_diff_us": sorted(diffs)[int(0.99 * (len(diffs) - 1))] if diffs else None}))


if __name__ == "__main__":
    main()
