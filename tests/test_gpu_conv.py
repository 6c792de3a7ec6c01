"""Implicit-GEMM convolutions (TMA im2col loads, no column matrix) against
the explicit im2col + GEMM path of the same kernels (bit-identical: same
tiles, same K order) and PyTorch fp32 conv2d (bf16 budget 1e-2 normwise),
in all three Tally shapes.  Needs a B200."""

from fractions import Fraction

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2410_07381_b200 as P
    from paper_2410_07381_b200 import kernels
    P.B200Device.get(0)
    return P, kernels, kernels.Stream(high_priority=False)


def _shapes(P, dk, s, out):
    res = []
    for shape in ("original", "sliced", "ptb"):
        out.zero_()
        ec = torch.zeros(dk.total_blocks, dtype=torch.int64, device="cuda")
        if shape == "original":
            dk.original(s, exec_count=ec).wait()
        elif shape == "sliced":
            for off, cnt in P.slice_plan(dk.total_blocks, Fraction(1, 3)):
                dk.sliced(s, off, cnt, exec_count=ec).wait()
        else:
            dk.ptb(s, 148, exec_count=ec).wait()
        assert bool((ec == 1).all()), shape
        res.append(out.clone())
    for r in res[1:]:
        assert torch.equal(r, res[0])
    return res[0]


def _rel(a, b):
    return ((a.double() - b.double()).abs().max() / b.double().abs().max()).item()


GEOMS = [  # n, h, w, c, cout, k, stride, pad
    (2, 14, 14, 64, 64, 3, 1, 1),
    (2, 16, 16, 128, 128, 3, 2, 1),
    (3, 8, 8, 256, 256, 3, 1, 1),
    (8, 14, 14, 256, 512, 1, 2, 0),
]


@pytest.mark.parametrize("geom", GEOMS)
def test_conv_fprop_matches_im2col_gemm_and_torch(env, geom):
    P, K, s = env
    n, h, w, c, cout, k, stride, pad = geom
    g = torch.Generator(device="cuda").manual_seed(sum(geom))
    x = (torch.randn(n, h, w, c, device="cuda", generator=g) * 0.5).bfloat16()
    wt = (torch.randn(cout, k * k * c, device="cuda", generator=g) * 0.05).bfloat16()   # (kh, kw, c) order
    ho, wo = (h + 2 * pad - k) // stride + 1, (w + 2 * pad - k) // stride + 1
    Pn = n * ho * wo
    y = torch.zeros(Pn, cout, device="cuda", dtype=torch.bfloat16)
    dk = K.conv_fprop(x, wt, y, n, h, w, c, k, stride, pad)
    out = _shapes(P, dk, s, y)
    # explicit path: im2col kernel + GEMM
    col = torch.zeros(Pn, k * k * c, device="cuda", dtype=torch.bfloat16)
    K.im2col(x, col, n, h, w, c, k, k, stride, pad).original(s).wait()
    y2 = torch.zeros_like(y)
    K.gemm(col, wt, y2).original(s).wait()
    assert torch.equal(out, y2)
    ref = torch.nn.functional.conv2d(x.float().permute(0, 3, 1, 2),
                                     wt.float().view(cout, k, k, c).permute(0, 3, 1, 2), stride=stride, padding=pad)
    assert _rel(out, ref.permute(0, 2, 3, 1).reshape(Pn, cout)) < 1e-2


@pytest.mark.parametrize("geom", GEOMS)
def test_conv_wgrad_matches_gemm_mn_and_torch(env, geom):
    P, K, s = env
    n, h, w, c, cout, k, stride, pad = geom
    g = torch.Generator(device="cuda").manual_seed(7 + sum(geom))
    x = (torch.randn(n, h, w, c, device="cuda", generator=g) * 0.5).bfloat16()
    ho, wo = (h + 2 * pad - k) // stride + 1, (w + 2 * pad - k) // stride + 1
    Pn = n * ho * wo
    dy = (torch.randn(Pn, cout, device="cuda", generator=g) * 0.5).bfloat16()
    kd = k * k * c
    S = 2
    part = torch.zeros(S, cout, kd, device="cuda")
    kb = (Pn + 63) // 64
    if (kb + (kb + S - 1) // S - 1) // ((kb + S - 1) // S) != S:
        S = 1
        part = torch.zeros(S, cout, kd, device="cuda")
    dk = K.conv_wgrad(dy, x, part, n, h, w, c, k, stride, pad, splits=S)
    out = _shapes(P, dk, s, part)
    col = torch.zeros(Pn, kd, device="cuda", dtype=torch.bfloat16)
    K.im2col(x, col, n, h, w, c, k, k, stride, pad).original(s).wait()
    part2 = torch.zeros_like(part)
    K.gemm_mn(dy, col, part2, splits=S).original(s).wait()
    assert torch.equal(out, part2)
    ref = dy.double().T @ col.double()
    assert _rel(out.sum(0), ref) < 1e-2


@pytest.mark.parametrize("geom", [(2, 14, 14, 64, 128, 3, 1, 1), (2, 8, 8, 256, 256, 3, 1, 1)])
def test_conv_dgrad_as_flipped_forward_conv(env, geom):
    """dx of a stride-1 'same' convolution as an implicit-GEMM forward
    convolution of dy with the flipped weight (ResNet50Train._flip), against
    PyTorch's conv2d input gradient."""
    P, K, s = env
    from paper_2410_07381_b200.resnet import ConvSpec, ResNet50Train
    n, h, w, c, cout, k, stride, pad = geom
    g = torch.Generator(device="cuda").manual_seed(3 + sum(geom))
    wt = (torch.randn(cout, k * k * c, device="cuda", generator=g) * 0.05)
    dy = (torch.randn(n * h * w, cout, device="cuda", generator=g) * 0.5).bfloat16()
    spec = ConvSpec("t", c, cout, k, stride, pad, h, w)
    wf = ResNet50Train._flip(wt, spec)
    dx = torch.zeros(n * h * w, c, device="cuda", dtype=torch.bfloat16)
    dk = K.conv_fprop(dy, wf, dx, n, h, w, cout, k, 1, k - 1 - pad)
    out = _shapes(P, dk, s, dx)
    x = torch.zeros(n, c, h, w, device="cuda", requires_grad=True)
    wr = wt.bfloat16().float().view(cout, k, k, c).permute(0, 3, 1, 2)
    y = torch.nn.functional.conv2d(x, wr, stride=stride, padding=pad)
    y.backward(dy.float().view(n, h, w, cout).permute(0, 3, 1, 2))
    ref = x.grad.permute(0, 2, 3, 1).reshape(n * h * w, c)
    assert _rel(out, ref) < 1e-2


STEM_GEOMS = [  # n, h, w, c (3 real channels padded to 8), cout, k, stride, pad -- the ResNet-50 stem
    (2, 32, 32, 8, 64, 7, 2, 3),
    (8, 30, 26, 8, 64, 7, 2, 3),   # (P = n*ho*wo a multiple of 8: the GEMM's K for the weight gradient)
    (2, 16, 16, 8, 64, 3, 1, 1),
]


def _stem_inputs(geom, seed):
    n, h, w, c, cout, k, stride, pad = geom
    g = torch.Generator(device="cuda").manual_seed(seed + sum(geom))
    x = (torch.randn(n, h, w, c, device="cuda", generator=g) * 0.5)
    x[..., 3:] = 0   # the stem's padding channels
    kd = k * k * c
    kp = (kd + 63) // 64 * 64
    wt = torch.zeros(cout, kp, device="cuda")
    wt[:, :kd] = torch.randn(cout, kd, device="cuda", generator=g) * 0.05
    return x.bfloat16(), wt.bfloat16(), kd, kp


@pytest.mark.parametrize("geom", STEM_GEOMS)
def test_conv_fprop_c8_matches_im2col_gemm(env, geom):
    """8-channel implicit convolution (one 16-byte im2col load per filter tap,
    no-swizzle operand layout) against im2col + GEMM (bit-identical) and
    PyTorch conv2d."""
    P, K, s = env
    n, h, w, c, cout, k, stride, pad = geom
    x, wt, kd, kp = _stem_inputs(geom, 11)
    ho, wo = (h + 2 * pad - k) // stride + 1, (w + 2 * pad - k) // stride + 1
    Pn = n * ho * wo
    y = torch.zeros(Pn, cout, device="cuda", dtype=torch.bfloat16)
    dk = K.conv_fprop(x, wt, y, n, h, w, c, k, stride, pad)
    assert dk.kind == "conv_fprop_c8_bf16_n64"
    out = _shapes(P, dk, s, y)
    col = torch.zeros(Pn, kp, device="cuda", dtype=torch.bfloat16)
    K.im2col(x, col, n, h, w, c, k, k, stride, pad).original(s).wait()
    y2 = torch.zeros_like(y)
    K.gemm(col, wt, y2).original(s).wait()
    assert torch.equal(out, y2)
    ref = torch.nn.functional.conv2d(x.float().permute(0, 3, 1, 2),
                                     wt[:, :kd].float().view(cout, k, k, c).permute(0, 3, 1, 2),
                                     stride=stride, padding=pad)
    assert _rel(out, ref.permute(0, 2, 3, 1).reshape(Pn, cout)) < 1e-2


@pytest.mark.parametrize("geom", STEM_GEOMS)
def test_conv_wgrad_c8_matches_gemm_mn(env, geom):
    P, K, s = env
    n, h, w, c, cout, k, stride, pad = geom
    x, _, kd, kp = _stem_inputs(geom, 5)
    ho, wo = (h + 2 * pad - k) // stride + 1, (w + 2 * pad - k) // stride + 1
    Pn = n * ho * wo
    g = torch.Generator(device="cuda").manual_seed(99)
    dy = (torch.randn(Pn, cout, device="cuda", generator=g) * 0.5).bfloat16()
    part = torch.zeros(1, cout, kp, device="cuda")
    dk = K.conv_wgrad(dy, x, part, n, h, w, c, k, stride, pad)
    assert dk.kind == "conv_wgrad_c8_bf16f32_n64"
    out = _shapes(P, dk, s, part)
    col = torch.zeros(Pn, kp, device="cuda", dtype=torch.bfloat16)
    K.im2col(x, col, n, h, w, c, k, k, stride, pad).original(s).wait()
    part2 = torch.zeros_like(part)
    K.gemm_mn(dy, col, part2).original(s).wait()
    assert torch.equal(out, part2)
    assert bool((out[0, :, kd:] == 0).all())   # padded taps: zero gradient
