"""Fixed cost of the PTB shape (diagnostics): ``spin`` kernels (each logical
block holds its slot for d ns, no memory traffic) launched Original and as
PTB with one worker per resident slot, for 1 and 4 blocks per worker; the
difference is the per-launch + per-block cost of the worker loop (first
claim, per-block claim/flag/barrier, retirement and outcome publication).

    python tools/ptb_fixed_cost.py
"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import kernels  # noqa: E402


def timed(launch, reps=20):
    ts = []
    for i in range(reps + 2):
        L = launch()
        L.wait()
        if i >= 2:
            ts.append(L.elapsed_ns)
    ts.sort()
    return ts[len(ts) // 2] / 1e3


def main():
    P.B200Device.get(0)
    s = kernels.Stream(high_priority=False)
    out = []
    for tpb in (256,):
        for d_ns in (0, 2000, 10000):
            for per in (1, 4):
                probe = kernels.spin(148, tpb, d_ns)
                occ = max(1, probe.info.occupancy_ptb)
                W = 148 * occ
                dk = kernels.spin(W * per, tpb, d_ns)
                o = timed(lambda: dk.original(s, timed=True))
                p = timed(lambda: dk.ptb(s, W, timed=True))
                out.append({"tpb": tpb, "block_us": d_ns / 1e3, "blocks_per_worker": per, "workers": W,
                            "original_us": o, "ptb_us": p, "ptb_minus_original_us": p - o})
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
