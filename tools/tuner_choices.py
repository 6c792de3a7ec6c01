"""The profile-guided tuner's choice for every best-effort kernel of a
configuration's training step (31.6 us threshold), with the candidate
records of the kernels it slices -- which kernels miss a preemptible PTB
configuration and why.

    python tools/tuner_choices.py [--config c4]
"""

from __future__ import annotations

import argparse
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2410_07381_b200 as P  # noqa: E402
from tools.ptb_overhead import program  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4", choices=["c2", "c3", "c4"])
    ap.add_argument("--threshold-us", type=float, default=31.6)
    args = ap.parse_args()
    dev = P.B200Device.get(0)
    tr = program(args.config)
    prof = P.Profiler(dev.spec, runs=3)
    hist = collections.Counter()
    sliced = {}
    for name, dk in tr.program:
        sig = tr.work_signature(name, dk)
        prof.bind(sig, dk)
        w = P.KernelWork(sig, dk.cost(), kernel=dk)
        c = prof.select(w.profile_key(), w.cost, int(args.threshold_us * 1000))
        hist[(dk.kind, c.variant)] += 1
        if c.variant == "Sliced" and sig not in sliced:
            recs = prof.profile(w.profile_key(), w.cost)
            sliced[sig] = {"name": name, "choice": c.describe(),
                           "records": [(r.candidate.describe(), r.kernel_latency_ns, r.turnaround_estimate_ns)
                                       for r in recs]}
    print(json.dumps({"config": args.config, "choices": {f"{k}:{v}": n for (k, v), n in sorted(hist.items())},
                      "sliced": sliced}, indent=1))


if __name__ == "__main__":
    main()
