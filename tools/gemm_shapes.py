"""tcgen05 GEMM shapes of the best-effort programs, timed alone (CUDA events
on the launch stream, L2 flushed before each launch): Original and PTB at
full occupancy, achieved TB/s (algorithmic bytes) and TFLOP/s.

    python tools/gemm_shapes.py [--only <label substring>]   # prints one JSON object

Environment knobs for experiments (read once per process by the library):
TALLY_GEMM_BLOCK_KB (k-blocks per logical block target), TALLY_GEMM_TPB_OLD.
"""

from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import kernels  # noqa: E402

# (label, M, N, K, out dtype): ResNet-50 bs=64 (C2) and transformer (C3/C4) shapes
SHAPES = [
    ("c2 layer2.0.conv1 fwd K=256", 200704, 128, 256, torch.bfloat16),
    ("c2 layer1 conv2 dgrad K=64", 200704, 576, 64, torch.bfloat16),
    ("c2 layer1 conv1 fwd K=64 N=64", 200704, 64, 64, torch.bfloat16),
    ("c2 layer1 conv3 fwd K=64 N=256", 200704, 256, 64, torch.bfloat16),
    ("c2 layer1 conv2 fwd K=576 N=64", 200704, 64, 576, torch.bfloat16),
    ("c2 layer3 conv3 fwd K=256 N=1024", 12544, 1024, 256, torch.bfloat16),
    ("c4 qkv fwd", 4096, 3072, 1024, torch.bfloat16),
    ("c3 fc fwd", 8192, 3072, 768, torch.bfloat16),
    ("square 8192", 8192, 8192, 8192, torch.bfloat16),
]


def main():
    P.B200Device.get(0)
    s = kernels.Stream(high_priority=False)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(0)
    out = {"env": {k: v for k, v in os.environ.items() if k.startswith("TALLY_GEMM")}}
    rows = []
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
    for label, M, N, K, dt in SHAPES:
        if only and only not in label:
            continue
        A = (torch.randn(M, K, device="cuda", generator=g) * 0.1).bfloat16()
        B = (torch.randn(N, K, device="cuda", generator=g) * 0.1).bfloat16()
        C = torch.empty(M, N, dtype=dt, device="cuda")
        dk = kernels.gemm(A, B, C)
        workers = dk.full_workers()

        def timed(fn, reps=5):
            ts = []
            for i in range(reps + 1):
                flush.zero_()
                L = fn()
                L.wait()
                if i:
                    ts.append(L.elapsed_ns)
            return sorted(ts)[len(ts) // 2]
        o = timed(lambda: dk.original(s, timed=True))
        ref = (A.float() @ B.float().t())
        err = ((C.float() - ref).abs().max() / ref.abs().max()).item()
        pt = timed(lambda: dk.ptb(s, workers, timed=True))
        i = dk.info
        rows.append({"shape": label, "kind": dk.kind, "blocks": dk.total_blocks, "ptb_workers": workers,
                     "orig_us": round(o / 1e3, 1), "ptb_us": round(pt / 1e3, 1),
                     "orig_TBps": round(i.alg_bytes / o / 1e3, 2), "orig_TFLOPs": round(i.alg_flops / o / 1e3, 1),
                     "ptb_TBps": round(i.alg_bytes / pt / 1e3, 2), "err": err})
        del A, B, C, dk
    out["rows"] = rows
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
