"""Config C3 workloads (BASELINE.json configs[2]): BERT-base inference (HP,
seq 128) next to GPT-2 small training (BE, bf16).

Best-effort training (``GPT2Train``) is one training step -- forward,
backward, momentum SGD -- written as a fixed program of this package's
transformable sm_100a kernels (like resnet.ResNet50Train): activations are
[tokens, channels] bf16 row-major matrices, statistics fp32.

  linear layer        gemm (x . W^T, W [out, in] bf16) -> bias_act (+ GELU / residual)
  attention           S = Q K^T and O = P V as batched gemm_ex over (sequence, head)
                      blocks of the fused QKV activation, softmax_causal in between
  LayerNorm           layernorm_fwd / layernorm_bwd (+ residual gradient) and
                      colstats for dgamma / dbeta
  backward            dX = dY . W reads W as stored (MN-major B); dW = dY^T . X
                      reads both activations as stored (MN-major A and B), split-K
  head                tied embedding: logits = LN(x) . wte^T (bf16), softmax_xent;
                      dX = dlogits . wte split-K (K = vocab) + splitk_reduce;
                      the wte gradient = head wgrad partials + an embedding
                      scatter slice (fp32 atomics), summed by sgd_update

Weights come from a HuggingFace ``GPT2LMHeadModel`` (random init -- no
checkpoints offline) so the parity tests compare against it.  The vocabulary
is padded to a multiple of 128 (zero rows; their gradient stays zero).
"""

from __future__ import annotations

from . import kernels as K
from .transformer import MOMENTUM, WEIGHT_DECAY, TransformerTrain, _pair_plan  # noqa: F401

LN_EPS = 1e-5


class GPT2Train(TransformerTrain):
    """One GPT-2 training step as a fixed sequence of device kernels.

    ``tokens`` [B, T] int32 input ids and ``targets`` [B*T] int32 next-token
    labels (refill between steps); ``loss`` [B*T] fp32 per-token losses."""

    gelu_act = 2          # GPT-2 "gelu_new" (tanh approximation)
    causal = True
    ln_eps = LN_EPS

    def __init__(self, batch=8, seq=1024, lr=1e-3, model=None, seed=0, device="cuda", n_layer=None):
        import torch
        if model is None:
            from transformers import GPT2Config, GPT2LMHeadModel
            torch.manual_seed(seed)
            cfg = GPT2Config(n_positions=max(1024, seq), resid_pdrop=0.0, embd_pdrop=0.0, attn_pdrop=0.0,
                             **({"n_layer": n_layer} if n_layer else {}))
            model = GPT2LMHeadModel(cfg)
        cfg = model.config
        self.ref_model = model
        self.B, self.T, self.d, self.H = batch, seq, cfg.n_embd, cfg.n_head
        self.D = self.d // self.H
        self.L = cfg.n_layer
        self.V = cfg.vocab_size
        self.Vp = (self.V + 127) // 128 * 128
        self.lr, self.device = lr, device
        if self.D != 64 or self.T % 128 or self.d % 128:
            raise ValueError("GPT2Train: head dim 64, seq and width multiples of 128")
        sd = {k: v.detach().float() for k, v in model.state_dict().items()}
        dev = device
        N, d = batch * seq, self.d
        self.N = N
        self._init_common()
        self.tokens = torch.zeros(batch, seq, dtype=torch.int32, device=dev)
        self.targets = torch.zeros(N, dtype=torch.int32, device=dev)
        self.loss = torch.zeros(N, dtype=torch.float32, device=dev)
        # embeddings (tied head)
        wte = torch.zeros(self.Vp, d, device=dev)
        wte[:self.V] = sd["transformer.wte.weight"].to(dev)
        self.wte = self._param("transformer.wte.weight", wte)
        self.wpe = self._param("transformer.wpe.weight", sd["transformer.wpe.weight"][:seq].to(dev).contiguous())
        self.layers = []
        for i in range(self.L):
            pre = f"transformer.h.{i}."
            lay = {"pre": pre}
            lay["ln1"] = self._ln(pre + "ln_1", sd)
            lay["qkv"] = self._linear(pre + "attn.c_attn", sd)
            lay["proj"] = self._linear(pre + "attn.c_proj", sd)
            lay["ln2"] = self._ln(pre + "ln_2", sd)
            lay["fc"] = self._linear(pre + "mlp.c_fc", sd)
            lay["fc2"] = self._linear(pre + "mlp.c_proj", sd)
            self.layers.append(lay)
        self.lnf = self._ln("transformer.ln_f", sd)
        self._build()
        self._finish(self.lr)

    def _linear(self, name, sd):
        """HF Conv1D (y = x W + b, W [in, out]) -> W [out, in] (y = x W^T)."""
        return self._linear_w(name, sd[name + ".weight"].t(), sd[name + ".bias"])

    def _ln(self, name, sd):
        return self._ln_w(name, sd[name + ".weight"], sd[name + ".bias"])

    # ---- the step ----------------------------------------------------------------------
    def _build(self):
        torch = self.torch
        N, d, T, H = self.N, self.d, self.T, self.H
        BHT = self.B * H * T
        # attention scratch shared by all layers (kernels run in order); P saved per layer
        S = torch.empty(BHT, T, dtype=torch.float32, device=self.device)
        dS = self._buf(BHT, T)
        x = self._buf(N, d)
        self._add("embedding", K.embedding_fwd(self.tokens.view(-1), self.wte.wb, self.wpe.wb, x, T))
        saved = []
        for i, lay in enumerate(self.layers):
            pre = lay["pre"]
            h1 = self._ln_fwd(pre + "ln_1", lay["ln1"], x)
            qkv = self._linear_fwd(pre + "attn.c_attn", lay["qkv"], h1)
            Pm = self._buf(BHT, T)
            o = self._attn_fwd(pre + "attn", qkv, S, Pm)
            x_mid = self._linear_fwd(pre + "attn.c_proj", lay["proj"], o, res=x)
            h2 = self._ln_fwd(pre + "ln_2", lay["ln2"], x_mid)
            hpre = self._buf(N, 4 * d)
            a = self._linear_fwd(pre + "mlp.c_fc", lay["fc"], h2, act=2, pre=hpre)
            x_next = self._linear_fwd(pre + "mlp.c_proj", lay["fc2"], a, res=x_mid)
            saved.append(dict(x=x, h1=h1, qkv=qkv, P=Pm, o=o, x_mid=x_mid, h2=h2, hpre=hpre, a=a))
            x = x_next
        self.x_final = x
        hf = self._ln_fwd("transformer.ln_f", self.lnf, x)
        logits = self._buf(N, self.Vp)
        pair_dec = _pair_plan(N, self.Vp, d, self.pair_gemms)[0]
        self._add("lm_head", K.gemm(hf, self.wte.wb, logits, pair=pair_dec))
        dl = self._buf(N, self.Vp)
        self._add("softmax_xent", K.softmax_xent(logits, None, self.targets, self.loss, dl, None, self.V))
        self.logits = logits
        # backward: head (tied wte: wgrad partials + one embedding-scatter slice)
        dhf = self._buf(N, d)
        self._gemm_ex_splitk("lm_head.dgrad", dl, self.wte.wb, dhf, N, d, self.Vp, b_mn=True)
        pw, Sw = _pair_plan(self.Vp, d, N, self.pair_gemms)
        self.wte.gpart = torch.zeros(Sw + 1, self.Vp, d, dtype=torch.float32, device=self.device)
        if Sw == 1:
            self._add("lm_head.wgrad", K.gemm_ex(dl, hf, self.wte.gpart[0], self.Vp, d, N, a_mn=True, b_mn=True, pair=pw))
        else:
            self._add("lm_head.wgrad", K.gemm_mn(dl, hf, self.wte.gpart[:Sw], splits=Sw, pair=pw))
        g = self._ln_bwd("transformer.ln_f", self.lnf, dhf, x)
        dP = torch.empty(BHT, T, dtype=torch.float32, device=self.device)
        self.block_grads = {}
        for lay, sv in zip(reversed(self.layers), reversed(saved)):
            pre = lay["pre"]
            da = self._linear_bwd(pre + "mlp.c_proj", lay["fc2"], g, sv["a"])
            du = self._buf(N, 4 * d)
            self._add(pre + "mlp.gelu_bwd", K.gelu_bwd(da, sv["hpre"], du))
            dh2 = self._linear_bwd(pre + "mlp.c_fc", lay["fc"], du, sv["h2"])
            dx_mid = self._ln_bwd(pre + "ln_2", lay["ln2"], dh2, sv["x_mid"], g2=g)
            do = self._linear_bwd(pre + "attn.c_proj", lay["proj"], dx_mid, sv["o"])
            dqkv = self._attn_bwd(pre + "attn", sv["qkv"], sv["P"], do, dP, dS)
            dh1 = self._linear_bwd(pre + "attn.c_attn", lay["qkv"], dqkv, sv["h1"])
            dx = self._ln_bwd(pre + "ln_1", lay["ln1"], dh1, sv["x"], g2=dx_mid)
            self.block_grads[pre] = dict(g=g, dx=dx)
            g = dx
        self.saved = saved
        # embeddings
        self._add("embedding.bwd", K.embedding_bwd(self.tokens.view(-1), g, self.wte.gpart[Sw]))
        self.sgd.add(self.wte.w, self.wte.v, self.wte.gpart, Sw + 1, self.Vp * d, WEIGHT_DECAY, self.wte.wb, None,
                     self.Vp, d, zero_from=Sw)
        self.wpe.g = torch.zeros(T * d, device=self.device)
        self._colsum("embedding.dwpe", g.view(self.B, T * d), self.wpe.g)
        self.sgd.add(self.wpe.w, self.wpe.v, self.wpe.g.view(1, -1), 1, T * d, WEIGHT_DECAY, self.wpe.wb, None, T, d)

    # ---- running it -------------------------------------------------------------------
    def set_batch(self, tokens):
        """tokens [B, T+1] int: inputs are tokens[:, :-1], targets tokens[:, 1:]."""
        self.tokens.copy_(tokens[:, :-1].to(self.torch.int32))
        self.targets.copy_(tokens[:, 1:].reshape(-1).to(self.torch.int32))


class BertInfer:
    """High-priority BERT-base inference request (HuggingFace, random init,
    bf16, batch 1) captured into one CUDA graph -- an unmodified application
    program launched as one exempt pipeline step."""

    def __init__(self, seq=128, seed=1, device="cuda"):
        import torch
        from transformers import BertConfig, BertModel
        torch.manual_seed(seed)
        m = BertModel(BertConfig()).eval().to(device=device, dtype=torch.bfloat16)
        self.model = m
        self.ids = torch.randint(0, 30522, (1, seq), device=device)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.no_grad():
            with torch.cuda.stream(side):
                for _ in range(3):
                    self.out = m(self.ids).last_hidden_state
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph):
                self.out = m(self.ids).last_hidden_state
        torch.cuda.synchronize()
        self.kernel = K.cuda_graph(self.graph)

    def reference(self):
        import torch
        with torch.no_grad():
            return self.model(self.ids).last_hidden_state
