"""Deterministic C2 launch sequences for ncu (no scheduler, no preemption).

    python tools/ncu_c2.py kernels [name ...]   # selected step kernels, Original then PTB
    python tools/ncu_c2.py step                 # one HP request + one full training step (Original)

Examples (under gpurun):
    ncu --set full --clock-control none -c 12 -o gpurun_out/ncu_c2 python tools/ncu_c2.py kernels
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv \\
        python tools/ncu_c2.py step
"""

from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import kernels, resnet  # noqa: E402

DEFAULT = ["layer3.0.conv2.gemm", "layer1.0.conv2.dgrad", "layer1.0.conv2.wgrad", "layer1.0.bn3.bwd",
           "layer1.0.bn3.bwd_stats", "conv1.im2col"]


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "kernels"
    P.B200Device.get(0)
    s = kernels.Stream(high_priority=False)
    tr = resnet.ResNet50Train(batch=64, image=224, lr=0.01)
    g = torch.Generator(device="cuda").manual_seed(0)
    tr.set_batch(torch.randn(64, 3, 224, 224, device="cuda", generator=g),
                 torch.randint(0, 1000, (64,), device="cuda", generator=g))
    if mode == "step":
        hp = resnet.ResNet50Infer(batch=1, image=224)
        hp.kernel.original(kernels.Stream(high_priority=True)).wait()
        tr.step_original(s)
    else:
        names = sys.argv[2:] or DEFAULT
        progs = dict(tr.program)
        for n in names:
            dk = progs[n]
            dk.original(s).wait()
            dk.ptb(s, dk.full_workers()).wait()
    torch.cuda.synchronize()
    print("ncu_c2 done:", mode)


if __name__ == "__main__":
    main()
