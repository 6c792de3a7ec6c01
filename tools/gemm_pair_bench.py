"""Single-CTA (128 x BN tiles, two CTAs per SM) vs CTA-pair (256 x 256 tiles,
cta_group::2, one CTA per SM) tcgen05 GEMMs against cuBLAS (torch.matmul), on
one B200: device time per launch (CUDA events on the launch stream, L2 flushed
before each launch, a spin kernel queued ahead so the events do not time the
host's launch latency), Original and PTB at the tuner's full-occupancy worker
count, TFLOP/s of 2*M*N*K.

    python tools/gemm_pair_bench.py [--only <label substring>] [--reps 5]
"""

from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import kernels  # noqa: E402

# (label, M, N, K, out dtype, splits)
SHAPES = [
    ("square 8192", 8192, 8192, 8192, torch.bfloat16, 1),
    ("square 4096", 4096, 4096, 4096, torch.bfloat16, 1),
    ("c4 qkv fwd", 4096, 3072, 1024, torch.bfloat16, 1),
    ("c4 ffn up fwd", 4096, 4096, 1024, torch.bfloat16, 1),
    ("c4 ffn down fwd (split 4)", 4096, 1024, 4096, torch.float32, 4),
    ("c4 ffn down fwd", 4096, 1024, 4096, torch.bfloat16, 1),
    ("c4 decoder fwd", 4096, 30720, 1024, torch.bfloat16, 1),
]


def main():
    P.B200Device.get(0)
    s = kernels.Stream(high_priority=False)
    # a ~30 us spin queued ahead of every timed launch: the launch and its
    # bracketing events are enqueued before the GPU reaches them, so the
    # events time the device, not the host's launch latency on an idle stream
    spin = kernels.spin(148, 32, 30_000)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(0)
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 5
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
    rows = []
    for label, M, N, K, dt, S in SHAPES:
        if only and only not in label:
            continue
        A = (torch.randn(M, K, device="cuda", generator=g) * 0.1).bfloat16()
        B = (torch.randn(N, K, device="cuda", generator=g) * 0.1).bfloat16()
        shape = (S, M, N) if S > 1 else (M, N)
        ref = (A.float() @ B.float().t())

        def timed(fn):
            ts = []
            for i in range(reps + 1):
                flush.zero_()
                torch.cuda.synchronize()
                spin.original(s)
                L = fn()
                L.wait()
                if i:
                    ts.append(L.elapsed_ns)
            return sorted(ts)[len(ts) // 2]

        row = {"shape": label, "M": M, "N": N, "K": K, "splits": S}
        flops = 2.0 * M * N * K
        for name, pair in (("single", False), ("pair", True)):
            C = torch.empty(*shape, dtype=dt, device="cuda")
            dk = kernels.gemm(A, B, C, splits=S, pair=pair)
            occ = max(1, dk.info.occupancy_ptb)
            workers = 148 * occ
            o = timed(lambda: dk.original(s, timed=True))
            cs = C.float().sum(0) if S > 1 else C.float()
            err = ((cs - ref).abs().max() / ref.abs().max()).item()
            pt = timed(lambda: dk.ptb(s, workers, timed=True))
            row[name] = {"kind": dk.kind, "blocks": dk.total_blocks, "ptb_workers": workers,
                         "orig_us": round(o / 1e3, 1), "ptb_us": round(pt / 1e3, 1),
                         "orig_TFLOPs": round(flops / o / 1e3, 1), "ptb_TFLOPs": round(flops / pt / 1e3, 1),
                         "err": err}
            dk.close()
            del C
        # cuBLAS (bf16 out, no split) on the default stream, CUDA events
        Cb = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        ts = []
        for i in range(reps + 1):
            flush.zero_()
            torch.cuda._sleep(60_000)   # same idea on torch's stream (~30 us)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(A, B.t(), out=Cb)
            e1.record()
            e1.synchronize()
            if i:
                ts.append(e0.elapsed_time(e1) * 1e6)
        cb = sorted(ts)[len(ts) // 2]
        row["cublas"] = {"us": round(cb / 1e3, 1), "TFLOPs": round(flops / cb / 1e3, 1)}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del A, B, ref
    print(json.dumps({"rows": rows}))


if __name__ == "__main__":
    main()
