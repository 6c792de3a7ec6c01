"""Deterministic launch sequences of a configuration's training step for ncu
(no scheduler, no preemption) -- the C2-C4 generalisation of ncu_c2.py.

    python tools/ncu_prog.py --config c4 step            # one full step, Original
    python tools/ncu_prog.py --config c4 kernels NAME..  # selected kernels, Original then PTB (full occupancy)
    python tools/ncu_prog.py --config c4 top             # print the step's largest launches

Examples (under gpurun):
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv \\
        python tools/ncu_prog.py --config c4 step
    ncu --set full --clock-control none -k regex:k_gemm -c 2 -o gpurun_out/ncu_c4_top \\
        python tools/ncu_prog.py --config c4 kernels cls.predictions.decoder.wgrad
"""

from __future__ import annotations

import argparse
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
    ap.add_argument("mode", choices=["step", "kernels", "top"])
    ap.add_argument("names", nargs="*")
    args = ap.parse_args()
    P.B200Device.get(0)
    s = kernels.Stream(high_priority=False)
    tr = program(args.config)
    if args.mode == "step":
        tr.step_original(s)
    elif args.mode == "top":
        tr.step_original(s)
        per = []
        for name, dk in tr.program:
            L = dk.original(s, timed=True)
            L.wait()
            per.append((L.elapsed_ns / 1e3, name, dk.kind))
        for us, name, kind in sorted(per, reverse=True)[:40]:
            print(f"{us:9.1f} us  {kind:20s} {name}")
    else:
        progs = dict(tr.program)
        for n in args.names:
            # exact name, else the first program entry containing it
            dk = progs[n] if n in progs else next(d for m, d in tr.program if n in m)
            dk.original(s).wait()
            dk.ptb(s, dk.full_workers()).wait()
    torch.cuda.synchronize()
    print("ncu_prog done:", args.config, args.mode)


if __name__ == "__main__":
    main()
