"""Transformation cost per kernel kind on the B200 (diagnostics, not the bench
contract): every kernel of a configuration's training step launched
untransformed and as PTB at full resident occupancy, each launch timed alone
with CUDA events behind a queued spin kernel (device time, not the host's
launch latency; L2 not flushed: the step's own order warms it), summed per
kind; PTB / Original time per kind is the inverse of the "transformed kernel
at >= 0.90 of untransformed" target.

    python tools/ptb_overhead.py [--config c2|c3|c4] [--reps 3] [--out FILE]
"""

from __future__ import annotations

import argparse
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import kernels  # noqa: E402


def program(config):
    g = torch.Generator(device="cuda").manual_seed(0)
    if config == "c2":
        from paper_2410_07381_b200 import resnet
        tr = resnet.ResNet50Train(batch=64, image=224)
        tr.set_batch(torch.randn(64, 3, 224, 224, device="cuda", generator=g),
                     torch.randint(0, 1000, (64,), device="cuda", generator=g))
    elif config == "c3":
        from paper_2410_07381_b200 import gpt2
        tr = gpt2.GPT2Train(batch=8, seq=1024)
        tr.set_batch(torch.randint(0, tr.V, (8, 1025), device="cuda", generator=g))
    else:
        from paper_2410_07381_b200 import bert
        tr = bert.BertTrain(batch=8, seq=512)
        tr.set_batch(torch.randint(0, tr.V, (8, 512), device="cuda", generator=g),
                     torch.randint(0, tr.V, (8, 512), device="cuda", generator=g))
    return tr


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4", choices=["c2", "c3", "c4"])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=None)
    ap.add_argument("--chosen", action="store_true", help="also time the tuner's chosen shape of every kernel")
    ap.add_argument("--launches", default=None, help="also write per-launch untransformed times (jsonl)")
    ap.add_argument("--no-spin", action="store_true",
                    help="time launches on an idle stream (the events then include the host's launch latency)")
    args = ap.parse_args()
    P.B200Device.get(0)
    s = kernels.Stream(high_priority=False)
    # a short spin queued ahead of every timed launch: the launch and its
    # events are enqueued before the GPU reaches them, so the events time the
    # device (as in a step, where the runtime keeps launches queued ahead)
    spin = kernels.spin(148, 32, 15_000)

    def ahead():
        if not args.no_spin:
            spin.original(s)
    tr = program(args.config)
    tr.step_original(s)
    tr.step_original(s)
    torch.cuda.synchronize()
    orig = collections.defaultdict(float)
    ptb = collections.defaultdict(float)
    n = collections.Counter()
    per = collections.defaultdict(float)
    alg_b = collections.defaultdict(float)
    alg_f = collections.defaultdict(float)
    for name, dk in tr.program:
        alg_b[dk.kind] += dk.info.alg_bytes
        alg_f[dk.kind] += dk.info.alg_flops
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                            "MEASURED_PEAKS.json")))
    except OSError:
        pass
    pk_t, pk_b = peaks.get("bf16_tflops", 1590.0), peaks.get("hbm_gbs", 6650.0)
    for _ in range(args.reps):
        for name, dk in tr.program:
            ahead()
            L = dk.original(s, timed=True)
            L.wait()
            orig[dk.kind] += L.elapsed_ns / 1e3 / args.reps
            per[name] += L.elapsed_ns / 1e3 / args.reps
            w = dk.full_workers()
            ahead()
            L = dk.ptb(s, w, timed=True)
            L.wait()
            ptb[dk.kind] += L.elapsed_ns / 1e3 / args.reps
    for name, dk in tr.program:
        n[dk.kind] += 1
    chosen = collections.defaultdict(float)
    if args.chosen:
        # the shapes the profile-guided tuner picks at the 31.6 us threshold
        from fractions import Fraction
        prof = P.Profiler(P.B200Device.get(0).spec, runs=3)
        for _ in range(args.reps):
            for name, dk in tr.program:
                sig = tr.work_signature(name, dk)
                prof.bind(sig, dk)
                w = P.KernelWork(sig, dk.cost(), kernel=dk)
                c = prof.select(w.profile_key(), w.cost, 31_600)
                ahead()
                if c.variant == "Ptb":
                    L = dk.ptb(s, c.worker_count, timed=True)
                    L.wait()
                    us = L.elapsed_ns / 1e3
                elif c.variant == "Sliced":
                    us = 0.0
                    for off, cnt in P.slice_plan(dk.total_blocks, Fraction(c.fraction)):
                        L = dk.sliced(s, off, cnt, timed=True)
                        L.wait()
                        us += L.elapsed_ns / 1e3
                else:
                    L = dk.original(s, timed=True)
                    L.wait()
                    us = L.elapsed_ns / 1e3
                chosen[dk.kind] += us / args.reps
    tot_o, tot_p = sum(orig.values()), sum(ptb.values())
    out = {"config": args.config, "kernels": len(tr.program), "step_us_original": tot_o, "step_us_ptb": tot_p,
           "peaks": {"bf16_tflops": pk_t, "hbm_gbs": pk_b, "source": "MEASURED_PEAKS.json" if peaks else
                     "fallback (B200_PROFILING.md)"},
           "ptb_vs_original_speed": tot_o / tot_p,
           "by_kind": {k: {"n": n[k], "original_us": round(orig[k], 1), "ptb_us": round(ptb[k], 1),
                           "speed_ratio": round(orig[k] / ptb[k], 3),
                           # roofline of the untransformed kind: algorithmic work over its device time
                           "alg_GB": round(alg_b[k] / 1e9, 3), "alg_GFLOP": round(alg_f[k] / 1e9, 1),
                           "achieved_TBps": round(alg_b[k] / (orig[k] * 1e3) / 1e3, 2),
                           "achieved_TFLOPs": round(alg_f[k] / (orig[k] * 1e3) / 1e3, 1),
                           "roofline_frac": round(max(alg_f[k] / (pk_t * 1e12), alg_b[k] / (pk_b * 1e9))
                                                  / (orig[k] * 1e-6), 3),
                           **({"chosen_us": round(chosen[k], 1), "chosen_speed_ratio": round(orig[k] / chosen[k], 3)}
                              if chosen else {})}
                       for k in sorted(orig, key=lambda k: -orig[k])}}
    if chosen:
        out["step_us_chosen"] = sum(chosen.values())
        out["chosen_vs_original_speed"] = tot_o / sum(chosen.values())
    if args.launches:
        with open(args.launches, "w") as f:
            for name, dk in tr.program:
                f.write(json.dumps({"name": name, "kind": dk.kind, "us": round(per[name], 2), "blocks": dk.total_blocks,
                                    "alg_MB": round(dk.info.alg_bytes / 1e6, 2),
                                    "alg_MFLOP": round(dk.info.alg_flops / 1e6, 1)}) + "\n")
    txt = json.dumps(out, indent=1)
    print(txt)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(txt)


if __name__ == "__main__":
    main()
