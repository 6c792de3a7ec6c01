"""Compare the B200 ResNet-50 training program's forward activations with the
PyTorch fp32 model layer by layer (debugging aid; needs a GPU)."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402
import torchvision  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import kernels, resnet  # noqa: E402


def nerr(x, ref):
    ref = ref.double()
    return ((x.double() - ref).abs().max() / ref.abs().max().clamp_min(1e-30)).item()


def main():
    P.B200Device.get(0)
    s = kernels.Stream(high_priority=False)
    torch.manual_seed(0)
    model = torchvision.models.resnet50(weights=None)
    B, img = 8, 64
    tr = resnet.ResNet50Train(batch=B, image=img, lr=0.05, model=model)
    g = torch.Generator(device="cuda").manual_seed(7)
    images = torch.randn(B, 3, img, img, device="cuda", generator=g).bfloat16()
    labels = torch.randint(0, 1000, (B,), device="cuda", generator=g)
    tr.set_batch(images, labels)
    # run the forward part only (up to softmax) to inspect
    for name, dk in tr.program:
        dk.original(s).wait()
        if name == "softmax_xent":
            break
    m = model.cuda().float().train()
    ref = {}

    def hook(name):
        def f(mod, inp, out):
            ref[name] = out.detach()
        return f
    m.conv1.register_forward_hook(hook("stem_conv"))
    m.relu.register_forward_hook(hook("stem"))
    m.maxpool.register_forward_hook(hook("maxpool"))
    for li in range(1, 5):
        for bi, blk in enumerate(getattr(m, f"layer{li}")):
            blk.register_forward_hook(hook(f"layer{li}.{bi}"))
    m.avgpool.register_forward_hook(hook("feat"))
    out = m(images.float())
    ref["logits"] = out
    for name, t in tr.acts.items():
        r = ref[name]
        if r.dim() == 4:
            r = r.permute(0, 2, 3, 1).reshape(-1, r.shape[1])
        else:
            r = r.reshape(t.shape[0], -1)
        tt = t[:, :r.shape[1]] if name == "logits" else t
        if name == "logits":
            tt = tt + tr.fc_b[:1000]
        print(f"{name:14s} shape {tuple(t.shape)} err {nerr(tt.reshape(r.shape), r):.3e}")
    print("loss ours", tr.loss.mean().item(), "ref", F.cross_entropy(out, labels).item())
    # the same model run by PyTorch in bf16: how far does plain bf16 drift?
    import copy
    mb = copy.deepcopy(m).bfloat16()
    refb = {}
    for li in range(1, 5):
        for bi, blk in enumerate(getattr(mb, f"layer{li}")):
            blk._forward_hooks.clear()
            blk.register_forward_hook(lambda mod, i, o, n=f"layer{li}.{bi}": refb.__setitem__(n, o.detach()))
    mb(images)
    for n in ("layer1.0", "layer2.0", "layer3.0", "layer4.0", "layer4.2"):
        print(f"torch-bf16 vs fp32 {n:10s} err {nerr(refb[n], ref[n]):.3e}")


if __name__ == "__main__" and "--train" not in sys.argv:
    main()


def train_trajectory(steps=12, lr=0.01, B=32, img=112):
    """Loss over repeated SGD steps on one fixed batch: our program vs the
    PyTorch fp32 model from the same initial weights (memorisation: both
    should fall)."""
    P.B200Device.get(0)
    s = kernels.Stream(high_priority=False)
    torch.manual_seed(0)
    model = torchvision.models.resnet50(weights=None)
    tr = resnet.ResNet50Train(batch=B, image=img, lr=lr, model=model)
    g = torch.Generator(device="cuda").manual_seed(7)
    images = torch.randn(B, 3, img, img, device="cuda", generator=g).bfloat16()
    labels = torch.randint(0, 1000, (B,), device="cuda", generator=g)
    tr.set_batch(images, labels)
    ours = []
    for _ in range(steps):
        tr.step_original(s)
        ours.append(round(tr.loss.mean().item(), 4))
    m = model.cuda().float().train()
    opt = torch.optim.SGD(m.parameters(), lr=lr, momentum=0.9, weight_decay=1e-4)
    ref = []
    for _ in range(steps):
        opt.zero_grad()
        loss = F.cross_entropy(m(images.float()), labels)
        ref.append(round(loss.item(), 4))
        loss.backward()
        opt.step()
    print("loss ours ", ours)
    print("loss torch", ref)


if __name__ == "__main__" and "--train" in sys.argv:
    train_trajectory()
