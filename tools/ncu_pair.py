"""One GEMM launch per (shape, kind, launch shape) for ncu captures of the
single-CTA and CTA-pair tcgen05 GEMMs (tools/gemm_pair_bench.py shapes).

    ncu --set full -k regex:k_gemm python tools/ncu_pair.py ffn_down qkv
"""

from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import kernels  # noqa: E402

SHAPES = {"ffn_down": (4096, 1024, 4096), "qkv": (4096, 3072, 1024), "square": (8192, 8192, 8192)}


def main():
    P.B200Device.get(0)
    s = kernels.Stream(high_priority=False)
    for name in sys.argv[1:] or ["ffn_down"]:
        M, N, K = SHAPES[name]
        A = (torch.randn(M, K, device="cuda") * 0.1).bfloat16()
        B = (torch.randn(N, K, device="cuda") * 0.1).bfloat16()
        C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        for pair in (False, True):
            dk = kernels.gemm(A, B, C, pair=pair)
            dk.original(s).wait()
            dk.ptb(s, 148 * max(1, dk.info.occupancy_ptb)).wait()
            dk.close()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
