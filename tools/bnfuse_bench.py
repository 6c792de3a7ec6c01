"""Fused batch-norm statistics in the GEMM / conv epilogue: device time per
launch with and without them, at the ResNet-50 (C2) producer shapes.
Spin-ahead CUDA events (device time), L2 flushed before each launch.

    [TALLY_BNFUSE_DBG=1|2] python tools/bnfuse_bench.py
"""
from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import kernels as K  # noqa: E402

SHAPES = [  # label, M, N, K, pair
    ("l1 conv3 x2", 200704, 256, 64, True),
    ("l1 conv1 n64", 200704, 64, 256, False),
    ("l2 conv1 128", 100352, 128, 256, False),
    ("l2 conv3 x2", 50176, 512, 128, True),
    ("l3 conv3 x2", 12544, 1024, 256, True),
]


def main():
    P.B200Device.get(0)
    s = K.Stream(high_priority=False)
    spin = K.spin(148, 32, 30_000)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(0)
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 6
    for label, M, N, Kd, pair in SHAPES:
        if only and only not in label:
            continue
        A = (torch.randn(M, Kd, device="cuda", generator=g) * 0.1).bfloat16()
        B = (torch.randn(N, Kd, device="cuda", generator=g) * 0.1).bfloat16()
        Y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        C = N
        bufs = [torch.zeros(C, device="cuda") for _ in range(4)] + [torch.zeros(2, C, device="cuda")]
        part = torch.zeros(K.BnStatsOut.part_floats(M, N, 32), device="cuda")
        bn = K.BnStatsOut(part, bufs[0], bufs[1], bufs[2], bufs[3], bufs[4], rb=int(os.environ.get("TALLY_BNFUSE_ROWS", "128")))
        out = {"label": label}
        for name, dk in (("plain", K.gemm(A, B, Y, pair=pair)), ("bn", K.gemm(A, B, Y, pair=pair, bn=bn))):
            ts = []
            for i in range(reps):
                flush.zero_()
                torch.cuda.synchronize()
                spin.original(s)
                L = dk.original(s, timed=True)
                L.wait()
                if i:
                    ts.append(L.elapsed_ns / 1e3)
            ts.sort()
            out[name] = round(ts[len(ts) // 2], 1)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
