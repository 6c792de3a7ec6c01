"""CTA-pair tcgen05 GEMMs (``*_x2`` kinds: a cluster of two SMs per 256 x 256
tile, ``tcgen05.mma.cta_group::2``, each CTA loading half of A and half of B)
in all three Tally shapes.  Needs a B200.

Tolerance (north star, bf16): max|C - C_ref| / max|C_ref| < 1e-2 against a
float64 reference of the same bf16 inputs; every shape (Original, Sliced,
PTB) bit-identical to the pair kernel's own Original launch and every logical
block executed exactly once.
"""

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


def _shapes(P, dk, stream, out, workers=(148, 296)):
    total = dk.total_blocks
    res = {}
    runs = [("original", None)] + [("sliced", f) for f in (Fraction(1, 3),)] + [("ptb", w) for w in workers]
    for name, arg in runs:
        out.zero_()
        ec = torch.zeros(total, dtype=torch.int64, device="cuda")
        if name == "original":
            dk.original(stream, exec_count=ec).wait()
        elif name == "sliced":
            for off, cnt in P.slice_plan(total, arg):
                dk.sliced(stream, off, cnt, exec_count=ec).wait()
        else:
            dk.ptb(stream, arg, exec_count=ec).wait()
        assert bool((ec == 1).all()), (name, arg)
        res[(name, arg)] = out.clone()
    base = res[("original", None)]
    for k, v in res.items():
        assert torch.equal(v, base), k
    return base


def _rel(c, ref):
    return ((c.double() - ref).abs().max() / ref.abs().max()).item()


@pytest.mark.parametrize("mnk", [(256, 256, 64), (1000, 512, 1024), (4096, 768, 1536)])
@pytest.mark.parametrize("out", ["bf16", "f32"])
def test_pair_gemm_kmajor(env, mnk, out):
    P, kernels, s = env
    M, N, K = mnk
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = (torch.rand(M, K, device="cuda", generator=g) * 2 - 1).bfloat16()
    B = (torch.rand(N, K, device="cuda", generator=g) * 2 - 1).bfloat16()
    C = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16 if out == "bf16" else torch.float32)
    dk = kernels.gemm(A, B, C, pair=True)
    assert dk.kind.endswith("_x2") and dk.info.cluster == 2
    c = _shapes(P, dk, s, C)
    assert _rel(c, A.double() @ B.double().T) < 1e-2
    # same math as the single-CTA kernel
    C1 = torch.zeros_like(C)
    d1 = kernels.gemm(A, B, C1)
    d1.original(s).wait()
    assert _rel(c, C1.double()) < 1e-2


def test_pair_gemm_splitk(env):
    P, kernels, s = env
    M, N, K, S = 1024, 512, 4096, 4
    g = torch.Generator(device="cuda").manual_seed(7)
    A = (torch.rand(M, K, device="cuda", generator=g) * 2 - 1).bfloat16()
    B = (torch.rand(N, K, device="cuda", generator=g) * 2 - 1).bfloat16()
    C = torch.zeros(S, M, N, device="cuda")
    dk = kernels.gemm(A, B, C, splits=S, pair=True)
    c = _shapes(P, dk, s, C)
    assert _rel(c.sum(0), A.double() @ B.double().T) < 1e-2


def test_pair_gemm_mn_weight_gradient(env):
    """dW = dY^T . X with both operands MN-major as stored (fp32, split-K)."""
    P, kernels, s = env
    T, M, N, S = 2048, 512, 768, 2
    g = torch.Generator(device="cuda").manual_seed(11)
    dY = (torch.rand(T, M, device="cuda", generator=g) * 2 - 1).bfloat16()
    X = (torch.rand(T, N, device="cuda", generator=g) * 2 - 1).bfloat16()
    C = torch.zeros(S, M, N, device="cuda")
    dk = kernels.gemm_mn(dY, X, C, splits=S, pair=True)
    c = _shapes(P, dk, s, C)
    assert _rel(c.sum(0), dY.double().T @ X.double()) < 1e-2


@pytest.mark.parametrize("out", ["bf16", "f32"])
def test_pair_gemm_kmn_batched(env, out):
    """P . V-like: A K-major, B MN-major, two batches at row offsets, strided C."""
    P, kernels, s = env
    Bt, M, N, K = 2, 512, 256, 512
    g = torch.Generator(device="cuda").manual_seed(13)
    A = (torch.rand(Bt * M, K, device="cuda", generator=g) * 2 - 1).bfloat16()
    Bm = (torch.rand(Bt * K, N + 256, device="cuda", generator=g) * 2 - 1).bfloat16()[:, :N]
    dt = torch.bfloat16 if out == "bf16" else torch.float32
    Cfull = torch.zeros(Bt * M, N + 128, device="cuda", dtype=dt)
    Cv = Cfull[:, :N]
    dk = kernels.gemm_ex(A, Bm, Cv, M, N, K, a_mn=False, b_mn=True, batches=Bt,
                         a_off=((M, 0), (0, 0)), b_off=((K, 0), (0, 0)), c_off=((M, 0), (0, 0)), pair=True)
    c = _shapes(P, dk, s, Cfull)
    for z in range(Bt):
        ref = A[z * M:(z + 1) * M].double() @ Bm[z * K:(z + 1) * K].double()
        assert _rel(c[z * M:(z + 1) * M, :N], ref) < 1e-2
    assert not c[:, N:].any()   # nothing outside the view


def test_pair_gemm_preempt_resume_exactly_once(env):
    """PTB pairs preempted by the counter trigger at several points, then
    resumed from the persisted counter: every tile exactly once, result equal
    to the uninterrupted run."""
    P, kernels, s = env
    M, N, K = 2048, 1024, 1024
    g = torch.Generator(device="cuda").manual_seed(17)
    A = (torch.rand(M, K, device="cuda", generator=g) * 2 - 1).bfloat16()
    B = (torch.rand(N, K, device="cuda", generator=g) * 2 - 1).bfloat16()
    C = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    dk = kernels.gemm(A, B, C, pair=True)
    dk.original(s).wait()
    ref = C.clone()
    total = dk.total_blocks
    for at in (1, 5, total // 2):
        C.zero_()
        ec = torch.zeros(total, dtype=torch.int64, device="cuda")
        st = dk.ptb(s, 16, preempt_at=at, exec_count=ec).wait()
        count = st.task_counter
        # blocks below the counter ran once or were handed back unrun (at
        # most one per worker pair: bounded retirement); none above it ran
        below = ec[:count].cpu().tolist()
        assert set(below) <= {0, 1} and below.count(0) <= 8
        assert bool((ec[count:] == 0).all())
        assert st.parked
        while not st.done:
            st = dk.ptb(s, 16, start_count=count, exec_count=ec).wait()
            count = st.task_counter
        assert bool((ec == 1).all()), at
        assert torch.equal(C, ref), at


def test_pair_ptb_rejects_odd_workers(env):
    P, kernels, s = env
    A = torch.zeros(256, 64, device="cuda", dtype=torch.bfloat16)
    B = torch.zeros(256, 64, device="cuda", dtype=torch.bfloat16)
    C = torch.zeros(256, 256, device="cuda", dtype=torch.bfloat16)
    dk = kernels.gemm(A, B, C, pair=True)
    with pytest.raises(Exception):
        dk.ptb(s, 3)


@pytest.mark.parametrize("pair", [False, True])
@pytest.mark.parametrize("act", [0, 2, 3])
def test_fused_linear_epilogue(env, pair, act):
    """y = act(x . W^T + b (+ res)) from the GEMM's TMA-store epilogue and the
    pre-activation beside it (bias_act semantics on the fp32 accumulator):
    against PyTorch fp32 of the same bf16 inputs within the bf16 budget, all
    shapes bit-identical."""
    P, kernels, s = env
    M, N, K = 1000, 512, 768
    g = torch.Generator(device="cuda").manual_seed(23 + act)
    x = (torch.rand(M, K, device="cuda", generator=g) * 2 - 1).bfloat16()
    w = (torch.rand(N, K, device="cuda", generator=g) * 2 - 1).bfloat16() * 0.05
    b = torch.rand(N, device="cuda", generator=g) - 0.5
    res = (torch.rand(M, N, device="cuda", generator=g) * 2 - 1).bfloat16()
    y = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    pre = torch.zeros_like(y)
    dk = kernels.gemm_ex(x, w, y, M, N, K, pair=pair, bias=b, res=res, pre=pre, act=act)
    outs = []
    for shape in ("original", "sliced", "ptb"):
        y.zero_()
        pre.zero_()
        if shape == "original":
            dk.original(s).wait()
        elif shape == "sliced":
            for off, cnt in P.slice_plan(dk.total_blocks, Fraction(1, 3)):
                dk.sliced(s, off, cnt).wait()
        else:
            dk.ptb(s, 148).wait()
        outs.append((y.clone(), pre.clone()))
    for o in outs[1:]:
        assert torch.equal(o[0], outs[0][0]) and torch.equal(o[1], outs[0][1])
    ref_pre = x.float() @ w.float().T + b + res.float()
    F = torch.nn.functional
    ref = {0: ref_pre, 2: F.gelu(ref_pre, approximate="tanh"), 3: F.gelu(ref_pre)}[act]
    assert _rel(outs[0][1], ref_pre.double()) < 1e-2
    assert _rel(outs[0][0], ref.double()) < 1e-2


def test_splitk_reduce_fused_epilogue(env):
    P, kernels, s = env
    S, M, N = 3, 512, 1024
    g = torch.Generator(device="cuda").manual_seed(29)
    parts = torch.randn(S, M, N, device="cuda", generator=g)
    b = torch.randn(N, device="cuda", generator=g)
    res = torch.randn(M, N, device="cuda", generator=g).bfloat16()
    y = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    pre = torch.zeros_like(y)
    dk = kernels.splitk_reduce(parts, y, bias=b, res=res, pre=pre, act=3)
    dk.original(s).wait()
    ref_pre = parts.sum(0) + b + res.float()
    assert _rel(pre, ref_pre.double()) < 1e-2
    assert _rel(y, torch.nn.functional.gelu(ref_pre).double()) < 1e-2
