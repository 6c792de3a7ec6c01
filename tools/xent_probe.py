"""softmax_xent at the GPT-2 LM-head shape (8192 rows x 50304 bf16 logits),
Original shape, for ncu:  ncu --set full -k regex:SoftmaxXent python tools/xent_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import kernels  # noqa: E402

P.B200Device.get(0)
B, V, Vp = 8192, 50257, 50304
g = torch.Generator(device="cuda").manual_seed(0)
logits = (torch.randn(B, Vp, device="cuda", generator=g) * 2).bfloat16()
labels = torch.randint(0, V, (B,), device="cuda", dtype=torch.int32, generator=g)
loss = torch.zeros(B, device="cuda")
dl = torch.empty(B, Vp, dtype=torch.bfloat16, device="cuda")
dk = kernels.softmax_xent(logits, None, labels, loss, dl, None, V)
s = kernels.Stream(high_priority=False)
for _ in range(3):
    L = dk.original(s, timed=True)
    L.wait()
print("softmax_xent us", L.elapsed_ns / 1e3, "info", dk.info)
