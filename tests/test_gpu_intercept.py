"""Generic best-effort routing: an unmodified PyTorch
training step (bf16 MLP + LayerNorm, MSE loss, momentum SGD) captured by
``intercept.capture`` -- its matmuls become transformable tcgen05 GEMMs, the
rest exempt CUDA-graph segments -- then run (a) untransformed in order and
(b) as the best-effort task of a Tally co-location with preemption; the
parameters track an eager PyTorch run of the same number of steps within the
bf16 tolerance.  Needs a B200."""

import copy

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _model(seed=0):
    torch.manual_seed(seed)
    m = torch.nn.Sequential(torch.nn.Linear(512, 2048), torch.nn.GELU(), torch.nn.Linear(2048, 512),
                            torch.nn.LayerNorm(512)).cuda().bfloat16()
    opt = torch.optim.SGD(m.parameters(), lr=0.05, momentum=0.9)
    return m, opt


def _step(m, opt, x, y):
    opt.zero_grad(set_to_none=False)
    loss = torch.nn.functional.mse_loss(m(x).float(), y)
    loss.backward()
    opt.step()


def _rel(a, b):
    return ((a.float() - b.float()).abs().max() / b.float().abs().max().clamp_min(1e-6)).item()


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2410_07381_b200 as P
    P.B200Device.get(0)
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(1024, 512, device="cuda", generator=g).bfloat16()
    y = torch.randn(1024, 512, device="cuda", generator=g)
    return P, x, y


def test_captured_step_matches_eager(env):
    P, x, y = env
    from paper_2410_07381_b200 import intercept, kernels
    m, opt = _model()
    ref_m = copy.deepcopy(m)
    ref_opt = torch.optim.SGD(ref_m.parameters(), lr=0.05, momentum=0.9)
    _step(m, opt, x, y)                 # warm the optimizer state (momentum buffers)
    _step(ref_m, ref_opt, x, y)
    prog = intercept.capture(_step, m, opt, x, y)      # eager step 2, recorded
    _step(ref_m, ref_opt, x, y)
    assert prog.n_gemm >= 5             # 2 forward + 3 backward matmuls (no grad for the input)
    kinds = {it[1].kind for it in prog.items if it[0] == "gemm"}
    assert any(k.startswith("gemm_bf16") for k in kinds)
    s = kernels.Stream(high_priority=False)
    for _ in range(3):                  # steps 3..5 through the program
        prog.run_original(s)
        _step(ref_m, ref_opt, x, y)
    torch.cuda.synchronize()
    for (n, p), rp in zip(m.named_parameters(), ref_m.parameters()):
        assert _rel(p, rp) < 2e-2, n


def test_captured_step_under_tally_with_preemption(env):
    """The captured program as the best-effort task of a Tally co-location
    (its GEMMs in the tuner's shapes, parked and resumed at HP arrivals):
    after n iterations the parameters are bit-identical to n untransformed
    in-order runs of the same program from the same state."""
    P, x, y = env
    from paper_2410_07381_b200 import intercept, kernels, workloads
    dev = P.B200Device.get(0)
    m, opt = _model(3)
    _step(m, opt, x, y)
    prog = intercept.capture(_step, m, opt, x, y)
    state = [p for p in m.parameters()] + [opt.state[p]["momentum_buffer"] for p in m.parameters()]
    snap = [t.detach().clone() for t in state]
    works = prog.works("mlp")
    g = torch.Generator(device="cuda").manual_seed(2)
    ha, hb, hc = (torch.rand(1 << 22, device="cuda", generator=g) for _ in range(3))
    hp = kernels.vecadd_f32(ha, hb, hc)
    prof = P.Profiler(dev.spec, runs=2)
    horizon = 40_000_000
    arr = workloads.generate_arrivals(0.3, 100_000, horizon, seed=4)
    tasks = [P.TaskScript("hp", P.HIGH, (P.KernelWork("vadd_hp", hp.cost(), kernel=hp),), arr),
             P.TaskScript("be", P.BEST_EFFORT, works)]
    res = P.run_policy(dev.spec, tasks, P.SchedulerConfig(policy="Tally"), horizon, profiler=prof,
                       record_events=False)
    torch.cuda.synchronize()
    n = len(res.iterations["be"])
    assert n >= 2 and len(res.requests["hp"]) == len(arr)
    assert torch.equal(hc, ha + hb)
    shapes = {r["shape"] for r in res.launches if r["task"] == 1}
    assert 2 in shapes, "no best-effort GEMM ran as PTB"
    after_tally = [t.detach().clone() for t in state]
    with torch.no_grad():
        for t, v in zip(state, snap):
            t.copy_(v)
    s = kernels.Stream(high_priority=False)
    for _ in range(n):
        prog.run_original(s)
    torch.cuda.synchronize()
    for i, (a, b) in enumerate(zip(after_tally, state)):
        assert torch.equal(a, b), (i, n)
