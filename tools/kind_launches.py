"""Per-launch device time of every C2 training-step kernel of the given
kinds (Original shape, L2 not flushed).  python tools/kind_launches.py bn_stats bn_stats_bwd"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import kernels, resnet  # noqa: E402


def main():
    kinds = set(sys.argv[1:])
    P.B200Device.get(0)
    s = kernels.Stream(high_priority=False)
    tr = resnet.ResNet50Train(batch=64, image=224, lr=0.01)
    g = torch.Generator(device="cuda").manual_seed(0)
    tr.set_batch(torch.randn(64, 3, 224, 224, device="cuda", generator=g),
                 torch.randint(0, 1000, (64,), device="cuda", generator=g))
    tr.step_original(s)
    for name, dk in tr.program:
        if dk.kind in kinds:
            L = dk.original(s, timed=True)
            L.wait()
            i = dk.info
            print(f"{name:32s} {dk.kind:14s} grid {i.grid} occ {i.occupancy_original} "
                  f"{L.elapsed_ns / 1e3:8.1f} us {i.alg_bytes / 1e6:8.1f} MB {i.alg_bytes / L.elapsed_ns:7.1f} GB/s")
        else:
            dk.original(s).wait()


if __name__ == "__main__":
    main()
