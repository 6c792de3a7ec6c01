"""Config C4 best-effort workload (BASELINE.json configs[3]): BERT-large
masked-LM training as a fixed program of this package's transformable
sm_100a kernels (the blocks of ``transformer.TransformerTrain``).

Post-LN encoder (HuggingFace ``BertForMaskedLM``, dropout off):

  embeddings   x0 = LN(wte[tok] + wpe[pos] + tte[0])          embedding_fwd, bias_act, layernorm_fwd
  layer        h1 = x + Attn(x) . Wo^T + bo ; x1 = LN(h1)      full (non-causal) softmax
               h2 = x1 + GELU(x1 W1^T + b1) W2^T + b2 ; x2 = LN(h2)   exact-erf GELU
  MLM head     t = LN(GELU(x Wt^T + bt)) ; logits = t . wte^T + bias (tied decoder, bf16)
               softmax_xent over every position (labels for all tokens)
  backward     the residual branches of the post-LN gradient are explicit adds
               (dx1 = dh2 + FFN'(dh2)); the decoder-bias gradient is a colstats
               column sum of dlogits; the wte gradient = decoder wgrad partials
               + one embedding-scatter slice, summed by sgd_update

Weights come from a HuggingFace ``BertForMaskedLM`` (random init) so the
parity test compares against it; Q, K, V are fused into one [3d, d] linear.
"""

from __future__ import annotations

from . import kernels as K
from .transformer import WEIGHT_DECAY, TransformerTrain, _pair_plan


class BertTrain(TransformerTrain):
    """One BERT masked-LM training step.  ``tokens`` [B, T] int32 inputs,
    ``labels`` [B*T] int32 targets (every position), ``loss`` [B*T] fp32."""

    gelu_act = 3          # BERT "gelu" (exact erf)
    causal = False

    def __init__(self, batch=8, seq=512, lr=1e-3, model=None, seed=0, device="cuda", n_layer=None, large=True):
        import torch
        if model is None:
            from transformers import BertConfig, BertForMaskedLM
            torch.manual_seed(seed)
            kw = dict(hidden_size=1024, num_hidden_layers=24, num_attention_heads=16, intermediate_size=4096) \
                if large else {}
            if n_layer:
                kw["num_hidden_layers"] = n_layer
            cfg = BertConfig(hidden_dropout_prob=0.0, attention_probs_dropout_prob=0.0,
                             max_position_embeddings=max(512, seq), **kw)
            model = BertForMaskedLM(cfg)
        cfg = model.config
        self.ref_model = model
        self.B, self.T, self.d, self.H = batch, seq, cfg.hidden_size, cfg.num_attention_heads
        self.D = self.d // self.H
        self.L = cfg.num_hidden_layers
        self.V = cfg.vocab_size
        self.Vp = (self.V + 255) // 256 * 256      # colstats (decoder-bias gradient) tiles 256 columns
        self.ln_eps = cfg.layer_norm_eps
        self.lr, self.device = lr, device
        if self.D != 64 or self.T % 128 or self.d % 128 or cfg.hidden_act != "gelu":
            raise ValueError("BertTrain: head dim 64, seq and width multiples of 128, erf GELU")
        sd = {k: v.detach().float() for k, v in model.state_dict().items()}
        dev = device
        N, d = batch * seq, self.d
        self.N = N
        self._init_common()
        self.tokens = torch.zeros(batch, seq, dtype=torch.int32, device=dev)
        self.labels = torch.zeros(N, dtype=torch.int32, device=dev)
        self.loss = torch.zeros(N, dtype=torch.float32, device=dev)
        e = "bert.embeddings."
        wte = torch.zeros(self.Vp, d, device=dev)
        wte[:self.V] = sd[e + "word_embeddings.weight"].to(dev)
        self.wte = self._param(e + "word_embeddings.weight", wte)
        self.wpe = self._param(e + "position_embeddings.weight",
                               sd[e + "position_embeddings.weight"][:seq].to(dev).contiguous())
        self.tte = self._param(e + "token_type_embeddings.weight", sd[e + "token_type_embeddings.weight"].to(dev),
                               bf16=False)
        self.ln_emb = self._ln(e + "LayerNorm", sd)
        self.layers = []
        for i in range(self.L):
            pre = f"bert.encoder.layer.{i}."
            a = pre + "attention."
            wqkv = torch.cat([sd[a + f"self.{n}.weight"] for n in ("query", "key", "value")])
            bqkv = torch.cat([sd[a + f"self.{n}.bias"] for n in ("query", "key", "value")])
            lay = {"pre": pre,
                   "qkv": self._linear_w(a + "self.qkv", wqkv, bqkv),
                   "proj": self._lin(a + "output.dense", sd),
                   "ln1": self._ln(a + "output.LayerNorm", sd),
                   "fc": self._lin(pre + "intermediate.dense", sd),
                   "fc2": self._lin(pre + "output.dense", sd),
                   "ln2": self._ln(pre + "output.LayerNorm", sd)}
            self.layers.append(lay)
        h = "cls.predictions."
        self.head = self._lin(h + "transform.dense", sd)
        self.ln_head = self._ln(h + "transform.LayerNorm", sd)
        dec_b = torch.zeros(self.Vp, device=dev)
        dec_b[:self.V] = sd[h + "bias"].to(dev)
        self.dec_b = self._param(h + "bias", dec_b, bf16=False)
        self._build()
        self._finish(self.lr)

    def _lin(self, name, sd):
        return self._linear_w(name, sd[name + ".weight"], sd[name + ".bias"])

    def _ln(self, name, sd):
        return self._ln_w(name, sd[name + ".weight"], sd[name + ".bias"])

    def _build(self):
        torch = self.torch
        N, d, T, H = self.N, self.d, self.T, self.H
        BHT = self.B * H * T
        # fp32 scores only for the unfused attention path (_fused_attn keeps them in TMEM)
        S = None if self._fused_attn() else torch.empty(BHT, T, dtype=torch.float32, device=self.device)
        dS = self._buf(BHT, T)
        # embeddings: word + position (embedding_fwd), + token type 0 (its fp32 row as the bias), LayerNorm
        e0 = self._buf(N, d)
        self._add("embeddings", K.embedding_fwd(self.tokens.view(-1), self.wte.wb, self.wpe.wb, e0, T))
        e1 = self._buf(N, d)
        self._add("embeddings.token_type", K.bias_act(e0, e1, self.tte.w[0], N, d))
        x = self._ln_fwd("embeddings.LayerNorm", self.ln_emb, e1)
        saved = []
        for lay in self.layers:
            pre = lay["pre"]
            qkv = self._linear_fwd(pre + "attention.self.qkv", lay["qkv"], x)
            Pm = self._buf(BHT, T)
            o = self._attn_fwd(pre + "attention.self", qkv, S, Pm)
            h1 = self._linear_fwd(pre + "attention.output.dense", lay["proj"], o, res=x)
            x1 = self._ln_fwd(pre + "attention.output.LayerNorm", lay["ln1"], h1)
            hpre = self._buf(N, lay["fc"].out)
            a = self._linear_fwd(pre + "intermediate.dense", lay["fc"], x1, act=self.gelu_act, pre=hpre)
            h2 = self._linear_fwd(pre + "output.dense", lay["fc2"], a, res=x1)
            x2 = self._ln_fwd(pre + "output.LayerNorm", lay["ln2"], h2)
            saved.append(dict(x=x, qkv=qkv, P=Pm, o=o, h1=h1, x1=x1, hpre=hpre, a=a, h2=h2))
            x = x2
        self.x_final = x
        # MLM head
        tpre = self._buf(N, d)
        t = self._linear_fwd("cls.predictions.transform.dense", self.head, x, act=self.gelu_act, pre=tpre)
        tl = self._ln_fwd("cls.predictions.transform.LayerNorm", self.ln_head, t)
        logits = self._buf(N, self.Vp)
        pair_dec = _pair_plan(N, self.Vp, d, self.pair_gemms)[0]
        self._add("cls.predictions.decoder", K.gemm(tl, self.wte.wb, logits, pair=pair_dec))
        dl = self._buf(N, self.Vp)
        self._add("softmax_xent", K.softmax_xent(logits, self.dec_b.w, self.labels, self.loss, dl, None, self.V))
        self.logits = logits
        # backward: decoder bias, tied decoder (dgrad split-K over the vocabulary, wgrad partials)
        self.dec_b.g = torch.zeros(self.Vp, device=self.device)
        self._colsum("cls.predictions.dbias", dl, self.dec_b.g)
        self.sgd.add(self.dec_b.w, self.dec_b.v, self.dec_b.g.view(1, -1), 1, self.Vp, WEIGHT_DECAY)
        dtl = self._buf(N, d)
        self._gemm_ex_splitk("cls.predictions.decoder.dgrad", dl, self.wte.wb, dtl, N, d, self.Vp, b_mn=True)
        pw, Sw = _pair_plan(self.Vp, d, N, self.pair_gemms)
        self.wte.gpart = torch.zeros(Sw + 1, self.Vp, d, dtype=torch.float32, device=self.device)
        if Sw == 1:
            self._add("cls.predictions.decoder.wgrad", K.gemm_ex(dl, tl, self.wte.gpart[0], self.Vp, d, N,
                                                                 a_mn=True, b_mn=True, pair=pw))
        else:
            self._add("cls.predictions.decoder.wgrad", K.gemm_mn(dl, tl, self.wte.gpart[:Sw], splits=Sw, pair=pw))
        dt = self._ln_bwd("cls.predictions.transform.LayerNorm", self.ln_head, dtl, t)
        du = self._buf(N, d)
        self._add("cls.predictions.transform.gelu_bwd", K.gelu_bwd(dt, tpre, du, erf=True))
        g = self._linear_bwd("cls.predictions.transform.dense", self.head, du, x)
        dP = None if self._fused_attn() else torch.empty(BHT, T, dtype=torch.float32, device=self.device)
        self.block_grads = {}
        for lay, sv in zip(reversed(self.layers), reversed(saved)):
            pre = lay["pre"]
            dh2 = self._ln_bwd(pre + "output.LayerNorm", lay["ln2"], g, sv["h2"])
            da = self._linear_bwd(pre + "output.dense", lay["fc2"], dh2, sv["a"])
            du = self._buf(N, lay["fc"].out)
            self._add(pre + "intermediate.gelu_bwd", K.gelu_bwd(da, sv["hpre"], du, erf=True))
            dx1 = self._linear_bwd(pre + "intermediate.dense", lay["fc"], du, sv["x1"], res=dh2)   # + residual grad
            dh1 = self._ln_bwd(pre + "attention.output.LayerNorm", lay["ln1"], dx1, sv["h1"])
            do = self._linear_bwd(pre + "attention.output.dense", lay["proj"], dh1, sv["o"])
            dqkv = self._attn_bwd(pre + "attention.self", sv["qkv"], sv["P"], do, dP, dS)
            dx = self._linear_bwd(pre + "attention.self.qkv", lay["qkv"], dqkv, sv["x"], res=dh1)
            self.block_grads[pre] = dict(g=g, dx=dx)
            g = dx
        self.saved = saved
        # embeddings backward: LayerNorm, then word (scatter slice), position and token-type sums
        ge = self._ln_bwd("embeddings.LayerNorm", self.ln_emb, g, e1)
        self._add("embeddings.word.bwd", K.embedding_bwd(self.tokens.view(-1), ge, self.wte.gpart[Sw]))
        self.sgd.add(self.wte.w, self.wte.v, self.wte.gpart, Sw + 1, self.Vp * d, WEIGHT_DECAY, self.wte.wb, None,
                     self.Vp, d, zero_from=Sw)
        self.wpe.g = torch.zeros(T * d, device=self.device)
        self._colsum("embeddings.position.bwd", ge.view(self.B, T * d), self.wpe.g)
        self.sgd.add(self.wpe.w, self.wpe.v, self.wpe.g.view(1, -1), 1, T * d, WEIGHT_DECAY, self.wpe.wb, None, T, d)
        self.tte.g = torch.zeros(self.tte.w.numel(), device=self.device)
        self._colsum("embeddings.token_type.bwd", ge, self.tte.g[:d])
        self.sgd.add(self.tte.w, self.tte.v, self.tte.g.view(1, -1), 1, self.tte.w.numel(), WEIGHT_DECAY)

    def set_batch(self, tokens, labels):
        """tokens [B, T], labels [B, T] (masked-LM targets, every position)."""
        self.tokens.copy_(tokens.to(self.torch.int32))
        self.labels.copy_(labels.reshape(-1).to(self.torch.int32))
