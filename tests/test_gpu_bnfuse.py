"""Batch-norm statistics fused into their producer (``csrc/bnfuse.cuh``):
the bf16 GEMM / implicit-GEMM convolution epilogue writes per-tile column
sums that ``bn_fold`` turns into mean, invstd and the bn_act scale / shift;
``splitk_reduce_bn`` does both in the split-K sum.

Checks, in all three Tally shapes (Original, Sliced, PTB), each logical block
exactly once:
* the output tensor is bit-identical to the same kernel without statistics;
* the statistics are bit-identical across shapes and worker counts (fixed
  fold order), and repeat launches (the chain counters reset themselves);
* they match float64 statistics of the stored bf16 output: mean within
  1e-5 * max|y|, invstd / scale / shift within 1e-4 relative (fp32 sums);
* rows past M (a 128-row tile tail) do not count.
Needs a B200.
"""

from fractions import Fraction

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
EPS = 1e-5


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2410_07381_b200 as P
    from paper_2410_07381_b200 import kernels
    P.B200Device.get(0)
    return P, kernels, kernels.Stream(high_priority=False)


def _bn_bufs(K, C, P, rb=128, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    gamma = torch.rand(C, device="cuda", generator=g) + 0.5
    beta = torch.rand(C, device="cuda", generator=g) - 0.5
    mean, invstd = torch.zeros(C, device="cuda"), torch.zeros(C, device="cuda")
    ss = torch.zeros(2, C, device="cuda")
    part = torch.zeros(K.BnStatsOut.part_floats(P, C, rb), device="cuda")
    return K.BnStatsOut(part, gamma, beta, mean, invstd, ss, EPS, rb), (gamma, beta, mean, invstd, ss)


def _check_stats(y, bufs):
    gamma, beta, mean, invstd, ss = bufs
    yd = y.double()
    m = yd.mean(0)
    var = (yd * yd).mean(0) - m * m
    isd = 1.0 / torch.sqrt(var.clamp_min(0) + EPS)
    scale = gamma.double() * isd
    shift = beta.double() - m * scale
    ymax = yd.abs().max().item()
    assert (mean.double() - m).abs().max().item() <= 1e-5 * ymax + 1e-7
    for got, ref in ((invstd, isd), (ss[0], scale)):
        assert ((got.double() - ref).abs() / ref.abs()).max().item() < 1e-4
    assert (ss[1].double() - shift).abs().max().item() < 1e-4 * (1 + shift.abs().max().item())


def _shapes(P, dk, s, out, bufs, workers=(148, 296)):
    """Run every shape; outputs and statistics bit-identical to Original."""
    res = []
    runs = [("original", None), ("original", None), ("sliced", Fraction(1, 3))] + [("ptb", w) for w in workers]
    for name, arg in runs:
        out.zero_()
        for b in bufs[2:]:
            b.zero_()
        ec = torch.zeros(dk.total_blocks, dtype=torch.int64, device="cuda")
        if name == "original":
            dk.original(s, exec_count=ec).wait()
        elif name == "sliced":
            for off, cnt in P.slice_plan(dk.total_blocks, arg):
                dk.sliced(s, off, cnt, exec_count=ec).wait()
        else:
            dk.ptb(s, arg, exec_count=ec).wait()
        assert bool((ec == 1).all()), (name, arg)
        res.append((out.clone(), [b.clone() for b in bufs[2:]]))
    for o, st in res[1:]:
        assert torch.equal(o, res[0][0])
        for a, b in zip(st, res[0][1]):
            assert torch.equal(a, b)
    return res[0][0]


def _fused_check(P, K, s, dk, Y, Y0, bn, bufs, M, N, rb=128):
    """The producer in every shape: output bit-identical to the unfused
    kernel, partial rows bit-identical across shapes; then bn_fold (every
    shape) -> statistics bit-identical and within tolerance of float64."""
    part = bn.tensors[0]
    R = K.BnStatsOut.gemm_rows(M, rb)
    rows = []
    for name, arg in [("original", None), ("sliced", Fraction(1, 3)), ("ptb", 148), ("ptb", 296)]:
        Y.zero_()
        part.fill_(float("nan"))
        ec = torch.zeros(dk.total_blocks, dtype=torch.int64, device="cuda")
        if name == "original":
            dk.original(s, exec_count=ec).wait()
        elif name == "sliced":
            for off, cnt in P.slice_plan(dk.total_blocks, arg):
                dk.sliced(s, off, cnt, exec_count=ec).wait()
        else:
            dk.ptb(s, arg, exec_count=ec).wait()
        assert bool((ec == 1).all()), (name, arg)
        assert torch.equal(Y, Y0), (name, arg)
        rows.append(part[:2 * R * N].clone())
    for r in rows[1:]:
        assert torch.equal(r, rows[0])
    assert not torch.isnan(rows[0]).any()
    fb, fbufs = _bn_bufs(K, N, R, rb=64, seed=0)
    fb2 = K.BnStatsOut(fb.tensors[0], *bufs, EPS, 64)
    fold = K.bn_fold(part, R, N, M, fb2)
    _shapes(P, fold, s, torch.zeros(1, device="cuda"), bufs)
    _check_stats(Y0, bufs)


@pytest.mark.parametrize("rb", [128, 32])
@pytest.mark.parametrize("mn", [(3136, 512, 256, False), (1000, 64, 128, False), (12544, 256, 1024, True),
                                (50176, 256, 64, False), (50176, 64, 64, False), (6272, 2048, 512, True)])
def test_gemm_bn_stats(env, mn, rb):
    P, K, s = env
    M, N, Kd, pair = mn
    g = torch.Generator(device="cuda").manual_seed(M + N)
    A = (torch.randn(M, Kd, device="cuda", generator=g) * 0.5).bfloat16()
    B = (torch.randn(N, Kd, device="cuda", generator=g) * 0.1 + 0.02).bfloat16()
    Y0 = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    K.gemm(A, B, Y0, pair=pair).original(s).wait()
    Y = torch.zeros_like(Y0)
    bn, bufs = _bn_bufs(K, N, 4 * M, seed=M, rb=rb)
    dk = K.gemm(A, B, Y, pair=pair, bn=bn)
    _fused_check(P, K, s, dk, Y, Y0, bn, bufs, M, N, rb)


@pytest.mark.parametrize("rb", [128, 32])
@pytest.mark.parametrize("geom", [(4, 14, 14, 64, 64, 3, 1, 1), (2, 16, 16, 128, 128, 3, 2, 1),
                                  (8, 7, 7, 256, 256, 3, 1, 1)])
def test_conv_fprop_bn_stats(env, geom, rb):
    P, K, s = env
    n, h, w, c, cout, k, stride, pad = geom
    g = torch.Generator(device="cuda").manual_seed(sum(geom))
    x = (torch.randn(n, h, w, c, device="cuda", generator=g)).bfloat16()
    W = (torch.randn(cout, k * k * c, device="cuda", generator=g) * 0.05).bfloat16()
    ho = (h + 2 * pad - k) // stride + 1
    Pn = n * ho * ho
    y0 = torch.zeros(Pn, cout, device="cuda", dtype=torch.bfloat16)
    K.conv_fprop(x, W, y0, n, h, w, c, k, stride, pad).original(s).wait()
    y1 = torch.zeros_like(y0)
    bn, bufs = _bn_bufs(K, cout, 4 * Pn, seed=n, rb=rb)
    dk = K.conv_fprop(x, W, y1, n, h, w, c, k, stride, pad, bn=bn)
    _fused_check(P, K, s, dk, y1, y0, bn, bufs, Pn, cout, rb)


@pytest.mark.parametrize("shape", [(3, 3136, 512), (2, 12544, 256), (5, 784, 2048), (1, 1000, 64), (4, 777, 128)])
def test_splitk_reduce_bn(env, shape):
    P, K, s = env
    S, Pn, C = shape
    g = torch.Generator(device="cuda").manual_seed(S * Pn + C)
    parts = torch.randn(S, Pn, C, device="cuda", generator=g) * 0.7 + 0.1
    y0 = torch.zeros(Pn, C, device="cuda", dtype=torch.bfloat16)
    K.splitk_reduce(parts, y0).original(s).wait()
    y1 = torch.zeros_like(y0)
    rb = 64
    bn, bufs = _bn_bufs(K, C, Pn, rb=rb, seed=S)
    dk = K.splitk_reduce_bn(parts, y1, bn)
    y = _shapes(P, dk, s, y1, bufs)
    assert torch.equal(y, y0)
    _check_stats(y, bufs)


def test_bn_stats_fused_rejects_split_output(env):
    P, K, s = env
    A = torch.zeros(256, 256, device="cuda", dtype=torch.bfloat16)
    B = torch.zeros(128, 256, device="cuda", dtype=torch.bfloat16)
    ws = torch.zeros(2, 256, 128, device="cuda")
    bn, _ = _bn_bufs(K, 128, 256)
    with pytest.raises(Exception, match="batch-norm"):
        K.gemm(A, B, ws, splits=2, bn=bn)
