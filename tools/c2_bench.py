"""Config C2 building blocks on the B200 (diagnostics, not the bench contract):

  * the ResNet-50 bs=64 training step as our kernel program, untransformed,
    back-to-back on one stream (device time, CUDA events) and its per-kind
    breakdown (each launch timed alone, L2 not flushed -- shares only);
  * the same step in PyTorch eager (cuDNN, bf16, channels-last) for scale;
  * the HP request: ResNet-50 bs=1 inference CUDA graph, solo latency;
  * the training step through the scheduler runtime (Eager policy, one BE
    task, untransformed) -- the per-kernel dispatch overhead.

    python tools/c2_bench.py [--batch 64] [--steps 5]
"""

from __future__ import annotations

import argparse
import collections
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import kernels, resnet  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--no-torch", action="store_true")
    args = ap.parse_args()
    dev = P.B200Device.get(0)
    out = {"batch": args.batch}
    s = kernels.Stream(high_priority=False)
    tr = resnet.ResNet50Train(batch=args.batch, image=224)
    g = torch.Generator(device="cuda").manual_seed(0)
    tr.set_batch(torch.randn(args.batch, 3, 224, 224, device="cuda", generator=g),
                 torch.randint(0, 1000, (args.batch,), device="cuda", generator=g))
    out["kernels_per_step"] = len(tr.program)
    for _ in range(2):
        tr.step_original(s)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    spans = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        launches = [dk.original(s) for _, dk in tr.program]
        for L in launches:
            L.wait()
        spans.append((time.perf_counter() - t0) * 1e3)
    spans.sort()
    out["step_ms_host_wall_median"] = spans[len(spans) // 2]
    out["loss"] = tr.loss.mean().item()
    # per-kind breakdown (each launch timed alone)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    per = []
    for name, dk in tr.program:
        L = dk.original(s, timed=True)
        L.wait()
        ns = L.elapsed_ns
        a = agg[dk.kind]
        a[0] += 1
        a[1] += ns / 1e3
        a[2] += dk.info.alg_bytes
        a[3] += dk.info.alg_flops
        per.append((ns / 1e3, name, dk.kind, dk.info.alg_bytes / max(ns, 1), dk.info.alg_flops / max(ns, 1) / 1e3))
    # the same, every kernel in PTB shape at full resident occupancy
    aggp = collections.defaultdict(lambda: [0, 0.0])
    for name, dk in tr.program:
        L = dk.ptb(s, dk.full_workers(), timed=True)
        L.wait()
        aggp[dk.kind][0] += 1
        aggp[dk.kind][1] += L.elapsed_ns / 1e3
    out["ptb_by_kind_us"] = {k: round(v[1], 1) for k, v in sorted(aggp.items(), key=lambda x: -x[1][1])}
    out["sum_of_kernel_us_ptb"] = sum(v[1] for v in aggp.values())
    tot = sum(a[1] for a in agg.values())
    out["sum_of_kernel_us"] = tot
    out["by_kind"] = {k: {"n": a[0], "us": round(a[1], 1), "share": round(a[1] / tot, 4),
                          "GBps": round(a[2] / (a[1] * 1e3), 1), "TFLOPs": round(a[3] / (a[1] * 1e6), 1)}
                      for k, a in sorted(agg.items(), key=lambda x: -x[1][1])}
    per.sort(reverse=True)
    out["top_launches"] = [{"us": round(u, 1), "name": n, "kind": k, "GBps": round(gb, 1), "TFLOPs": round(tf, 1)}
                           for u, n, k, gb, tf in per[:25]]
    # PyTorch eager bf16 channels-last training step for scale
    if not args.no_torch:
        import torchvision
        m = torchvision.models.resnet50(weights=None).cuda().to(memory_format=torch.channels_last).bfloat16()
        opt = torch.optim.SGD(m.parameters(), lr=0.1, momentum=0.9, weight_decay=1e-4)
        xb = torch.randn(args.batch, 3, 224, 224, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
        yb = torch.randint(0, 1000, (args.batch,), device="cuda")
        for i in range(3 + args.steps):
            if i == 3:
                torch.cuda.synchronize()
                ev0.record()
            opt.zero_grad(set_to_none=True)
            torch.nn.functional.cross_entropy(m(xb), yb).backward()
            opt.step()
        ev1.record()
        torch.cuda.synchronize()
        out["torch_eager_bf16_step_ms"] = ev0.elapsed_time(ev1) / args.steps
        del m, opt
    # HP request: inference graph solo
    hp = resnet.ResNet50Infer(batch=1, image=224)
    hs = kernels.Stream(high_priority=True)
    lat = []
    for i in range(30):
        L = hp.kernel.original(hs, timed=True)
        L.wait()
        if i >= 5:
            lat.append(L.elapsed_ns / 1e3)
    lat.sort()
    out["hp_infer_us_median"] = lat[len(lat) // 2]
    # through the runtime: Eager, BE only
    prof = P.Profiler(dev.spec, runs=1)
    works = []
    for name, dk in tr.program:
        sig = tr.work_signature(name, dk)
        prof.bind(sig, dk)
        works.append(P.KernelWork(sig, dk.cost(), kernel=dk))
    be = P.TaskScript("be", P.BEST_EFFORT, tuple(works))
    res = P.run_policy(dev.spec, [be], P.SchedulerConfig(policy="Eager"), int(1e9), profiler=prof,
                       record_events=False)
    it = res.iterations["be"]
    if len(it) >= 2:
        gaps = [b - a for a, b in zip(it, it[1:])]
        out["runner_eager_step_ms"] = sorted(gaps)[len(gaps) // 2] / 1e6
    out["runner_iterations_1s"] = len(it)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
