"""Short, deterministic launch sequence for ncu captures (no preemption, no
daemon): each kind once in Original shape, then once in PTB shape.

    ncu --set full -k regex:k_gemm ... python tools/ncu_target.py sgemm_tf32x3
"""

from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import kernels  # noqa: E402
from tools.microbench import make  # noqa: E402


def main():
    kinds = sys.argv[1:] or ["sgemm_tf32x3"]
    P.B200Device.get(0)
    s = kernels.Stream(high_priority=False)
    for kind in kinds:
        dk = make(kind)
        workers = 148 * min(4, dk.info.occupancy_ptb)
        dk.original(s).wait()
        dk.ptb(s, workers).wait()
    torch.cuda.synchronize()
    print("ncu_target done:", " ".join(kinds))


if __name__ == "__main__":
    main()
