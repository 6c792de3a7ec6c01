"""Best-effort training program alone through the runtime (run_policy) at
several look-ahead depths, against the program back to back on one stream
-- how much of the native step the real-time dispatch keeps.

    python tools/lookahead_probe.py [--config c4] [--ms 3000] [--policy Eager|Tally]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import kernels  # noqa: E402
from tools.ptb_overhead import program  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4", choices=["c2", "c3", "c4"])
    ap.add_argument("--ms", type=float, default=3000.0)
    ap.add_argument("--policy", default="Eager")
    ap.add_argument("--depths", default="1,4,8,16")
    args = ap.parse_args()
    dev = P.B200Device.get(0)
    tr = program(args.config)
    s = kernels.Stream(high_priority=False)
    for _ in range(3):
        tr.step_original(s)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 10
    for _ in range(n):
        tr.step_original(s)
    torch.cuda.synchronize()
    native = n / (time.perf_counter() - t0)
    prof = P.Profiler(dev.spec, runs=3)
    works = []
    for name, dk in tr.program:
        sig = tr.work_signature(name, dk)
        prof.bind(sig, dk)
        works.append(P.KernelWork(sig, dk.cost(), kernel=dk))
    task = P.TaskScript("be", P.BEST_EFFORT, tuple(works))
    cfg = P.SchedulerConfig(policy=args.policy)
    window = int(args.ms * 1e6)
    out = {"config": args.config, "policy": args.policy, "native_steps_per_s": native, "runtime": {}}
    for L in (int(x) for x in args.depths.split(",")):
        res = P.run_policy(dev.spec, [task], cfg, window, profiler=prof, record_events=False,
                           options={"lookahead": L})
        warm = window // 10
        done = sum(1 for t in res.iterations["be"] if t >= warm)
        out["runtime"][str(L)] = done / ((window - warm) / 1e9)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
