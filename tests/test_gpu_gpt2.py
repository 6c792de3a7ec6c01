"""Config C3 best-effort training (GPT-2) and its transformer kernels on a
B200: each kernel against a PyTorch fp32 reference in all three Tally shapes
(bit-identical to each other), and one training step of a 2-layer GPT-2
against HuggingFace GPT2LMHeadModel (fp32 autograd) on the same weights.

Tolerances, normwise max|x - ref| / max|ref|: bf16-output kernels 1e-2;
fp32 statistics 1e-4; the training step's loss and every parameter gradient
1e-2 end to end (measured worst 9.8e-3, the tied embedding: GELU and softmax
are smooth, so unlike the ResNet step no ReLU masks flip and an end-to-end
comparison holds)."""

from fractions import Fraction

import pytest

torch = pytest.importorskip("torch")
F = pytest.importorskip("torch.nn.functional")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2410_07381_b200 as P
    from paper_2410_07381_b200 import kernels
    P.B200Device.get(0)
    return P, kernels, kernels.Stream(high_priority=False)


def nerr(x, ref):
    ref = ref.double()
    return ((x.double() - ref).abs().max() / ref.abs().max().clamp_min(1e-30)).item()


def shapes(P, dk, stream, outs):
    res = {}
    total = dk.total_blocks
    workers = 148 * min(2, max(1, dk.info.occupancy_ptb))
    for shape in ("original", "sliced", "ptb"):
        for o in outs:
            o.zero_()
        ec = torch.zeros(total, dtype=torch.int64, device="cuda")
        if shape == "original":
            dk.original(stream, exec_count=ec).wait()
        elif shape == "sliced":
            for off, cnt in P.slice_plan(total, Fraction(1, 5)):
                dk.sliced(stream, off, cnt, exec_count=ec).wait()
        else:
            dk.ptb(stream, min(workers, total), exec_count=ec).wait()
        assert bool((ec == 1).all()), shape
        res[shape] = [o.clone() for o in outs]
    for a, b, c in zip(res["original"], res["sliced"], res["ptb"]):
        assert torch.equal(a, b) and torch.equal(a, c)
    return res["original"]


def rnd(*shape, seed=0, dtype=torch.bfloat16, scale=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(*shape, device="cuda", generator=g) * scale).to(dtype)


def test_layernorm_fwd_bwd_and_param_grads(env):
    P, kernels, stream = env
    N, C = 300, 768
    x = (rnd(N, C, seed=1).float() * 2 + 0.3).bfloat16()
    gamma = torch.rand(C, device="cuda") + 0.5
    beta = torch.randn(C, device="cuda")
    y = torch.zeros_like(x)
    mean, rstd = torch.zeros(N, device="cuda"), torch.zeros(N, device="cuda")
    gy, gm, gr = shapes(P, kernels.layernorm_fwd(x, y, gamma, beta, mean, rstd), stream, [y, mean, rstd])
    xf = x.float().requires_grad_(True)
    gmf, btf = gamma.clone().requires_grad_(True), beta.clone().requires_grad_(True)
    ref = F.layer_norm(xf, (C,), gmf, btf, eps=1e-5)
    assert nerr(gy, ref) < 1e-2 and nerr(gm, xf.mean(1)) < 1e-5
    mean.copy_(gm)
    rstd.copy_(gr)
    dy, g2 = rnd(N, C, seed=2), rnd(N, C, seed=3)
    ref.backward(dy.float())
    dx = torch.zeros_like(x)
    (gdx,) = shapes(P, kernels.layernorm_bwd(dy, x, gamma, mean, rstd, dx, g2=g2), stream, [dx])
    assert nerr(gdx, xf.grad + g2.float()) < 1e-2
    dg, db = torch.zeros(C, device="cuda"), torch.zeros(C, device="cuda")
    part = torch.zeros(2 * 10 * C, device="cuda")
    gdg, gdb = shapes(P, kernels.colstats(dy, part, N, C, 32, db, dgamma=dg, x=x, mean=mean, rstd=rstd), stream,
                      [dg, db])
    assert nerr(gdg, gmf.grad) < 1e-4 and nerr(gdb, btf.grad) < 1e-4


@pytest.mark.parametrize("erf", [False, True])     # GPT-2 tanh approximation / BERT exact erf
def test_bias_gelu_and_backward(env, erf):
    P, kernels, stream = env
    N, C = 200, 3072
    u, bias = rnd(N, C, seed=4), torch.randn(C, device="cuda")
    y, pre = torch.zeros_like(u), torch.zeros_like(u)
    gy, gp = shapes(P, kernels.bias_act(u, y, bias, N, C, act=3 if erf else 2, pre=pre), stream, [y, pre])
    h = (u.float() + bias).requires_grad_(True)
    ref = F.gelu(h, approximate="none" if erf else "tanh")
    assert nerr(gy, ref) < 1e-2 and nerr(gp, h) < 1e-2
    g = rnd(N, C, seed=5)
    ref.backward(g.float())
    dx = torch.zeros_like(u)
    (gdx,) = shapes(P, kernels.gelu_bwd(g, gp, dx, erf=erf), stream, [dx])
    assert nerr(gdx, h.grad) < 2e-2


@pytest.mark.parametrize("causal", [True, False])   # GPT-2 / BERT encoder
def test_softmax_causal_fwd_bwd(env, causal):
    P, kernels, stream = env
    BH, T = 6, 256
    S = torch.randn(BH * T, T, device="cuda") * 3
    Pm = torch.zeros(BH * T, T, dtype=torch.bfloat16, device="cuda")
    scale = 0.125
    (gp,) = shapes(P, kernels.softmax_causal(S, Pm, T, scale, causal=causal), stream, [Pm])
    mask = torch.ones(T, T, device="cuda").tril().bool() if causal else torch.ones(T, T, device="cuda").bool()
    s3 = (S.view(BH, T, T) * scale).masked_fill(~mask, float("-inf")).requires_grad_(True)
    ref = torch.softmax(s3, -1)
    assert nerr(gp.view(BH, T, T), ref) < 1e-2
    dP = torch.randn(BH * T, T, device="cuda")
    ref.backward(dP.view(BH, T, T))
    dS = torch.zeros_like(Pm)
    (gds,) = shapes(P, kernels.softmax_causal_bwd(gp, dP, dS, T, scale, causal=causal), stream, [dS])
    # reference from the bf16 probabilities the program keeps (d/dS of softmax(scale*S))
    pf = gp.float().view(BH, T, T)
    dref = pf * (dP.view(BH, T, T) - (pf * dP.view(BH, T, T)).sum(-1, keepdim=True)) * scale
    assert nerr(gds.view(BH, T, T), dref) < 1e-2
    assert nerr(gds.view(BH, T, T), s3.grad.masked_fill(~mask, 0) * scale) < 3e-2


def test_embedding_fwd_bwd(env):
    P, kernels, stream = env
    V, T, C, B = 1000, 128, 768, 2
    wte, wpe = rnd(V, C, seed=6), rnd(T, C, seed=7)
    tok = torch.randint(0, V, (B * T,), device="cuda", dtype=torch.int32)
    x = torch.zeros(B * T, C, dtype=torch.bfloat16, device="cuda")
    (gx,) = shapes(P, kernels.embedding_fwd(tok, wte, wpe, x, T), stream, [x])
    ref = wte.float()[tok.long()] + wpe.float().repeat(B, 1)
    assert nerr(gx, ref) < 1e-2
    dx = rnd(B * T, C, seed=8)
    dw = torch.zeros(V, C, device="cuda")
    kernels.embedding_bwd(tok, dx, dw).ptb(stream, 148).wait()
    refw = torch.zeros(V, C, device="cuda").index_add_(0, tok.long(), dx.float())
    assert nerr(dw, refw) < 1e-5


def _small_model():
    from transformers import GPT2Config, GPT2LMHeadModel
    torch.manual_seed(0)
    cfg = GPT2Config(n_layer=2, n_positions=128, resid_pdrop=0.0, embd_pdrop=0.0, attn_pdrop=0.0)
    return GPT2LMHeadModel(cfg)


def test_gpt2_train_step_vs_huggingface(env):
    P, kernels, stream = env
    from paper_2410_07381_b200 import gpt2
    model = _small_model()
    B, T, lr = 2, 128, 1e-2
    tr = gpt2.GPT2Train(batch=B, seq=T, lr=lr, model=model)
    g = torch.Generator(device="cuda").manual_seed(3)
    toks = torch.randint(0, tr.V, (B, T + 1), device="cuda", generator=g)
    tr.set_batch(toks)
    w0 = {name: t.clone() for name, t in tr.params}
    tr.step_original(stream)
    loss = tr.loss.mean().item()
    m = model.cuda().float().train()
    m.zero_grad()
    logits = m(toks[:, :-1]).logits
    ref_loss = F.cross_entropy(logits.reshape(-1, tr.V), toks[:, 1:].reshape(-1))
    ref_loss.backward()
    assert abs(loss - ref_loss.item()) / ref_loss.item() < 1e-2, (loss, ref_loss.item())
    hf = dict(m.named_parameters())
    errs = {}
    for name, t in tr.params:
        gr_ours = (w0[name] - t) / lr          # momentum buffer starts at 0, weight decay 0
        key = name if name in hf else "lm_head.weight"
        ref = hf[key].grad
        if name.endswith(".weight") and ("c_attn" in name or "c_proj" in name or "c_fc" in name):
            ref = ref.t()
        if name == "transformer.wte.weight":
            gr_ours = gr_ours[:tr.V]
        if name == "transformer.wpe.weight":
            ref = ref[:T]
        errs[name] = nerr(gr_ours, ref)
    for k, v in errs.items():
        print(f"gpt2-grad {k} {v:.3e}")
    bad = {k: v for k, v in errs.items() if v > 1e-2}
    assert not bad, bad


def test_gpt2_step_shapes_bit_identical(env):
    """Every kernel of the step in PTB / Sliced shape gives the untransformed
    result (the wte gradient's embedding scatter uses fp32 atomics: 1e-6)."""
    P, kernels, stream = env
    from paper_2410_07381_b200 import gpt2
    outs = {}
    for shape in ("original", "ptb", "sliced"):
        tr = gpt2.GPT2Train(batch=2, seq=128, lr=1e-2, model=_small_model())
        g = torch.Generator(device="cuda").manual_seed(5)
        tr.set_batch(torch.randint(0, tr.V, (2, 129), device="cuda", generator=g))
        for name, dk in tr.program:
            if shape == "original":
                dk.original(stream).wait()
            elif shape == "ptb":
                dk.ptb(stream, dk.full_workers()).wait()
            else:
                for off, cnt in P.slice_plan(dk.total_blocks, Fraction(1, 4)):
                    dk.sliced(stream, off, cnt).wait()
        outs[shape] = {n: t.clone() for n, t in tr.params}
        outs[shape]["loss"] = tr.loss.clone()
    for n in outs["original"]:
        a, b, c = outs["original"][n], outs["ptb"][n], outs["sliced"][n]
        if n == "transformer.wte.weight":
            assert nerr(b, a) < 1e-6 and nerr(c, a) < 1e-6
        else:
            assert torch.equal(a, b) and torch.equal(a, c), n


def test_bert_infer_graph(env):
    P, kernels, stream = env
    from paper_2410_07381_b200 import gpt2
    hp = gpt2.BertInfer(seq=128)
    hs = kernels.Stream(high_priority=True)
    hp.kernel.original(hs).wait()
    # graph replay vs eager of the same bf16 model: cuDNN/SDPA may pick other
    # kernels under capture (measured 1.8e-2 normwise)
    assert nerr(hp.out, hp.reference()) < 5e-2
