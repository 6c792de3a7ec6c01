"""Config C3 building blocks on the B200 (diagnostics): the GPT-2 small
training step (batch 8, seq 1024) as our kernel program -- back-to-back step
time, per-kind breakdown (Original and PTB), PyTorch eager bf16 for scale --
and the BERT-base seq-128 inference graph's solo latency.

    python tools/c3_bench.py [--batch 8] [--no-torch]
"""

from __future__ import annotations

import collections
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import gpt2, kernels  # noqa: E402


def main():
    B = int(sys.argv[sys.argv.index("--batch") + 1]) if "--batch" in sys.argv else 8
    P.B200Device.get(0)
    s = kernels.Stream(high_priority=False)
    tr = gpt2.GPT2Train(batch=B, seq=1024, lr=1e-3)
    g = torch.Generator(device="cuda").manual_seed(0)
    tr.set_batch(torch.randint(0, tr.V, (B, 1025), device="cuda", generator=g))
    out = {"batch": B, "kernels_per_step": len(tr.program)}
    losses = []
    for _ in range(3):
        tr.step_original(s)
        losses.append(round(tr.loss.mean().item(), 4))
    spans = []
    for _ in range(5):
        t0 = time.perf_counter()
        tr.step_original(s)
        spans.append((time.perf_counter() - t0) * 1e3)
        losses.append(round(tr.loss.mean().item(), 4))
    out["step_ms_host_wall_median"] = sorted(spans)[2]
    out["loss_trajectory"] = losses
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0.0])
    for name, dk in tr.program:
        L = dk.original(s, timed=True)
        L.wait()
        a = agg[dk.kind]
        a[0] += 1
        a[1] += L.elapsed_ns / 1e3
        a[2] += dk.info.alg_flops
        Lp = dk.ptb(s, dk.full_workers(), timed=True)
        Lp.wait()
        a[3] += Lp.elapsed_ns / 1e3
        a[4] += dk.info.alg_bytes
    tot = sum(a[1] for a in agg.values())
    out["sum_of_kernel_us"] = tot
    out["sum_of_kernel_us_ptb"] = sum(a[3] for a in agg.values())
    out["by_kind"] = {k: {"n": a[0], "us": round(a[1], 1), "ptb_us": round(a[3], 1), "share": round(a[1] / tot, 4),
                          "TFLOPs": round(a[2] / (a[1] * 1e6), 1), "GBps": round(a[4] / (a[1] * 1e3), 1)}
                      for k, a in sorted(agg.items(), key=lambda x: -x[1][1])}
    if "--no-torch" not in sys.argv:
        from transformers import GPT2Config, GPT2LMHeadModel
        m = GPT2LMHeadModel(GPT2Config()).cuda().bfloat16()
        opt = torch.optim.SGD(m.parameters(), lr=1e-3, momentum=0.9)
        x = torch.randint(0, 50257, (B, 1025), device="cuda")
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for i in range(6):
            if i == 2:
                torch.cuda.synchronize()
                ev0.record()
            opt.zero_grad(set_to_none=True)
            lo = m(x[:, :-1], labels=x[:, :-1]).loss
            lo.backward()
            opt.step()
        ev1.record()
        torch.cuda.synchronize()
        out["torch_eager_bf16_step_ms"] = ev0.elapsed_time(ev1) / 4
        del m, opt
    hp = gpt2.BertInfer(seq=128)
    hs = kernels.Stream(high_priority=True)
    lat = []
    for i in range(30):
        L = hp.kernel.original(hs, timed=True)
        L.wait()
        if i >= 5:
            lat.append(L.elapsed_ns / 1e3)
    out["hp_bert_us_median"] = sorted(lat)[len(lat) // 2]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
