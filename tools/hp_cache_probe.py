"""Why is the HP request slower next to the BE job?  Times the ResNet-50 bs=1
inference graph (device time, CUDA events) after different predecessors:

  warm       back-to-back requests
  l2flush    after writing 512 MB (evicts L2, keeps TLB mostly warm)
  be_step    after a full ResNet-50 bs=64 training step (L2 + TLB + icache)
  be_kernel  after one large BE kernel (layer1 bn_bwd, ~100 MB)

with and without the L2-persisting window on the HP weights.

    python tools/hp_cache_probe.py
"""

from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import kernels, resnet  # noqa: E402


def med(xs):
    s = sorted(xs)
    return round(s[len(s) // 2] / 1e3, 1)


def main():
    P.B200Device.get(0)
    be_s = kernels.Stream(high_priority=False)
    hp_s = kernels.Stream(high_priority=True)
    tr = resnet.ResNet50Train(batch=64, image=224, lr=0.01)
    g = torch.Generator(device="cuda").manual_seed(0)
    tr.set_batch(torch.randn(64, 3, 224, 224, device="cuda", generator=g),
                 torch.randint(0, 1000, (64,), device="cuda", generator=g))
    big = next(dk for name, dk in tr.program if name == "layer1.0.bn3.bwd")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    out = {"l2_MB": torch.cuda.get_device_properties(0).L2_cache_size / 2 ** 20}
    try:
        from cuda.bindings import runtime as rt
        err, v = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, 0)
        out["max_persisting_l2_MB"] = v / 2 ** 20
    except Exception as e:   # noqa: BLE001
        out["max_persisting_l2_MB"] = repr(e)
    spin = kernels.spin(148 * 8, 256, 100_000)   # 100 us of pure SM occupancy, no memory traffic
    sweep = torch.empty(12 << 30, dtype=torch.uint8, device="cuda")   # 12 GB, touched once per 2 MB page
    gemm = next(dk for name, dk in tr.program if name == "layer3.0.conv2.gemm")
    for persist, warm in ((None, False), ("nodes", False), (None, True), ("nodes", True)):
        hp = resnet.ResNet50Infer(batch=1, image=224, persist_l2=persist, warm_l2=warm)
        res = {"l2_window_MB": hp.l2_window_bytes / 2 ** 20}
        for label in ("warm", "flush64", "be_kernel", "be_gemm", "be_step"):
            ts = []
            for i in range(12):
                if label == "l2flush":
                    flush.zero_()
                elif label == "flush64":
                    flush[:64 << 20].zero_()
                elif label == "be_kernel":
                    big.original(be_s).wait()
                elif label == "be_kernel_sleep2ms":
                    big.original(be_s).wait()
                    import time as _t
                    t_end = _t.perf_counter() + 0.002
                    while _t.perf_counter() < t_end:
                        pass
                elif label == "be_kernel_then_hp":
                    big.original(be_s).wait()
                    hp.kernel.original(hp_s).wait()
                elif label == "tlb_sweep":
                    sweep[:: 2 << 20].zero_()      # ~6000 pages, 6 KB of data
                elif label == "spin100us":
                    spin.original(be_s).wait()
                elif label == "be_gemm":
                    gemm.original(be_s).wait()
                elif label == "be_step":
                    tr.step_original(be_s)
                torch.cuda.synchronize()
                L = hp.kernel.original(hp_s, timed=True)
                L.wait()
                if i >= 2:
                    ts.append(L.elapsed_ns)
            res[label] = med(ts)
        out[f"persist={persist} warm={warm}"] = res
        del hp
        torch.cuda.synchronize()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
