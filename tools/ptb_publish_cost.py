"""Timing experiment: what the host-visible outcome publication costs a PTB
launch.  Run once with the normal build and once with
TALLY_NVCC_DEFINES=-DTALLY_EXPERIMENT_NO_MIRROR (launches then never report
completion: timed with their CUDA events after a device synchronize).

    python tools/ptb_publish_cost.py
"""

import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import _lib, kernels  # noqa: E402


def elapsed(L):
    torch.cuda.synchronize()
    v = C.c_longlong()
    _lib.check(_lib.lib.tally_launch_elapsed_ns(L.id, C.byref(v)), "elapsed")
    return v.value / 1e3


def main():
    P.B200Device.get(0)
    s = kernels.Stream(high_priority=False)
    out = {}
    for d in (0, 10000):
        dk = kernels.spin(1184, 256, d)
        po = []
        for i in range(14):
            Lp = dk.ptb(s, 1184, timed=True)
            tp = elapsed(Lp)
            Lo = dk.original(s, timed=True)
            to = elapsed(Lo)
            if i >= 4:
                po.append((tp, to))
        po.sort()
        out[f"block_us={d / 1e3}"] = {"ptb_us": po[len(po) // 2][0], "original_us": po[len(po) // 2][1]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
