"""Kernel-shape microbenchmarks on the B200 (not the bench contract; see bench.py).

    python tools/microbench.py [--kind vecadd_f32|rowsum_f32|sgemm_tf32x3|gemm_bf16]

Prints one JSON object: per-shape device time (CUDA events around each
launch, L2 flushed in between), achieved GB/s or TFLOP/s, and preemption
latency for both flag placements.
"""

from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import kernels  # noqa: E402


def make(kind):
    g = torch.Generator(device="cuda").manual_seed(0)
    if kind == "vecadd_f32":
        n = 1 << 24
        a, b, c = (torch.rand(n, device="cuda", generator=g) for _ in range(3))
        return kernels.vecadd_f32(a, b, c)
    if kind == "rowsum_f32":
        x = torch.rand(1 << 16, 1024, device="cuda", generator=g)
        return kernels.rowsum_f32(x, torch.zeros(1 << 16, device="cuda"))
    if kind.startswith("sgemm_tf32x3"):
        m = 4096
        A = torch.rand(m, m, device="cuda", generator=g) * 2 - 1
        B = torch.rand(m, m, device="cuda", generator=g) * 2 - 1
        sg = kernels.sgemm_tf32x3(A, B, torch.zeros(m, m, device="cuda"),
                                  tile_n=64 if kind.endswith("n64") else 128)
        sg.prepare(kernels.Stream(high_priority=False))
        sg.gemm._owner = sg
        return sg.gemm
    if kind == "gemm_bf16":
        m = 8192
        A = (torch.rand(m, m, device="cuda", generator=g) * 2 - 1).bfloat16()
        B = (torch.rand(m, m, device="cuda", generator=g) * 2 - 1).bfloat16()
        return kernels.gemm_bf16(A, B, torch.zeros(m, m, device="cuda", dtype=torch.bfloat16))
    raise SystemExit(f"unknown kind {kind}")


def main():
    kind = sys.argv[sys.argv.index("--kind") + 1] if "--kind" in sys.argv else "vecadd_f32"
    dev = P.B200Device.get(0)
    dk = make(kind)
    s = kernels.Stream(high_priority=False)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    info = dk.info
    out = {"kind": kind, "gpu": dev.name, "stream_mem_ops": dev.stream_mem_ops,
           "stream_mem_ops_probe": dev.info.stream_mem_ops_probe,
           "total_blocks": info.total_blocks,
           "occupancy_ptb": info.occupancy_ptb, "alg_bytes": info.alg_bytes,
           "alg_flops": info.alg_flops, "shapes": {}}

    def timed(fn, reps=10):
        ts = []
        for _ in range(3):
            fn().wait()
        for _ in range(reps):
            flush.zero_()
            torch.cuda.synchronize()
            ts.append(fn().elapsed_ns)
        ts.sort()
        return ts[len(ts) // 2]

    shapes = {"original": lambda: dk.original(s, timed=True)}
    for k in (1, 2, 4, 8):
        if k <= info.occupancy_ptb:
            w = 148 * k
            shapes[f"ptb{w}"] = lambda w=w: dk.ptb(s, w, timed=True)
    for name, fn in shapes.items():
        t = timed(fn)
        rec = {"ns": t}
        if info.alg_bytes:
            rec["GBps"] = info.alg_bytes / t
        if info.alg_flops:
            rec["TFLOPs"] = info.alg_flops / t / 1e3
        out["shapes"][name] = rec
    # flag propagation: host signal -> a spinning device reader sees it
    import ctypes as C
    from paper_2410_07381_b200 import _lib
    out["flag_propagation_us"] = {}
    for mode, name in ((0, "device_streamwrite"), (1, "host_mapped")):
        med, mx = C.c_longlong(), C.c_longlong()
        if _lib.lib.tally_probe_flag_latency(mode, 20, C.byref(med), C.byref(mx)) == 0:
            out["flag_propagation_us"][name] = {"median": med.value / 1e3, "max": mx.value / 1e3}
    # preemption latency, both flag placements
    off, unc = dev.clock_offset()
    out["clock_uncertainty_ns"] = unc
    for mode in ("device", "host"):
        if mode == "device" and not dev.stream_mem_ops:
            continue
        dev.set_flag_mode(mode == "host")
        lats, drains = [], []
        nw = 148 * min(4, info.occupancy_ptb)
        wlog = torch.zeros(nw, 4, dtype=torch.int64, device="cuda")
        for k in range(12):
            L = dk.ptb(s, nw, worker_log=wlog)
            t = P.B200Device.now_ns() + 10_000 + 3_000 * k
            while P.B200Device.now_ns() < t:
                pass
            L.preempt()
            st = L.wait()
            if st.parked:
                lats.append(st.gt_last_exit + off - st.host_preempt_ns)
                drains.append(st.gt_last_exit - st.gt_first_stop)
                if k == 0:
                    w = wlog.cpu()
                    entry = (w[:, 1] - w[:, 1].min()) / 1e3
                    exit_ = (w[:, 2] - st.host_preempt_ns + off) / 1e3
                    done = w[:, 0] & 0xffffffff
                    out[f"workers_{mode}"] = {
                        "entry_us_min_med_max": [float(entry.min()), float(entry.median()), float(entry.max())],
                        "exit_after_signal_us_min_med_max": [float(exit_.min()), float(exit_.median()), float(exit_.max())],
                        "blocks_min_med_max": [int(done.min()), int(done.median()), int(done.max())],
                        "stopped": int(w[:, 3].sum()), "distinct_sms": int(len(set((w[:, 0] >> 32).tolist())))}
        lats.sort()
        drains.sort()
        if lats:
            out[f"preempt_{mode}_flag"] = {"n": len(lats), "median_us": lats[len(lats) // 2] / 1e3,
                                           "max_us": lats[-1] / 1e3,
                                           "drain_median_us": drains[len(drains) // 2] / 1e3}
    dev.set_flag_mode(not dev.stream_mem_ops)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
