"""Back-to-back untransformed training step of a configuration's best-effort
program on one stream (no scheduler): device time per step with CUDA events
-- the 'native' ceiling of the BE throughput, for A/B experiments
(environment knobs such as TALLY_CARVEOUT=max).

    python tools/step_time.py [--config c4] [--steps 5]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import kernels  # noqa: E402
from tools.ptb_overhead import program  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4", choices=["c2", "c3", "c4"])
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    P.B200Device.get(0)
    s = kernels.Stream(high_priority=False)
    tr = program(args.config)
    for _ in range(3):
        tr.step_original(s)
    torch.cuda.synchronize()
    ext = torch.cuda.ExternalStream(s.handle())
    times = []
    for _ in range(args.steps):
        if ext is not None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ext)
            tr.step_original(s)
            e1.record(ext)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        else:
            import time
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            tr.step_original(s)
            torch.cuda.synchronize()
            times.append((time.perf_counter() - t0) * 1e3)
    times.sort()
    print(json.dumps({"config": args.config, "env": {k: v for k, v in os.environ.items() if k.startswith("TALLY_")},
                      "kernels": len(tr.program), "step_ms_median": times[len(times) // 2], "step_ms": times}))


if __name__ == "__main__":
    main()
