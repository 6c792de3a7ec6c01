"""Shared building blocks of the transformer best-effort training programs
(configs C3 and C4: ``gpt2.GPT2Train``, ``bert.BertTrain``).

A program is a fixed list of this package's transformable sm_100a kernels
(every one launchable Original / Sliced / PTB), run strictly in order by the
scheduler.  Activations are [tokens, channels] bf16 row-major matrices,
statistics and master weights fp32, one momentum-SGD ``sgd_update`` over a
segment table of all parameters at the end.

  linear layer   gemm (x . W^T, W [out, in] bf16) -> bias_act (+ GELU / residual)
  attention      S = Q K^T and O = P V as batched gemm_ex over (sequence, head)
                 blocks of the fused QKV activation, softmax in between
                 (causal for GPT-2, full for BERT)
  LayerNorm      layernorm_fwd / layernorm_bwd (+ residual gradient) and
                 colstats for dgamma / dbeta
  backward       dX = dY . W reads W as stored (MN-major B); dW = dY^T . X reads
                 both activations as stored (MN-major A and B), split-K fp32
                 partials summed by sgd_update
"""

from __future__ import annotations

import math
import os

from . import kernels as K
from .resnet import SgdTable, _gemm_splits, _pair_plan  # noqa: F401

MOMENTUM = 0.9
WEIGHT_DECAY = 0.0


def _rb_cols(P, C):
    """Rows per colstats logical block (~128 KB of gradient per block)."""
    base = 1024 if C < 128 else (512 if C < 256 else 256)
    cblocks = (C + 255) // 256
    target = int(os.environ.get("TALLY_COLSTATS_BLOCKS", "296"))   # experiment knob
    return max(8, min(base, P * cblocks // target // 8 * 8))


class TransformerTrain:
    """Base: parameter bookkeeping and the layer building blocks.

    Subclasses set ``B, T, d, H, D, N, device, ln_eps, gelu_act, causal``,
    call ``_init_common()`` first and ``_finish()`` after adding their
    kernels."""

    gelu_act = 2          # bias_act activation code: 2 GELU tanh, 3 GELU erf
    causal = True
    ln_eps = 1e-5
    pair_gemms = True     # CTA-pair tcgen05 GEMMs for the large linear layers (_pair_plan)
    fuse_attention = os.environ.get("TALLY_FUSE_ATTENTION", "1") != "0"   # see _fused_attn
    # which linear-layer epilogues run fused in the GEMM (or split-K reduce):
    # "bias" (bias only), "res" (bias + residual), "act" (bias + activation).
    # Measured (tools/step_time.py, BERT-large step): none 27.5 ms, bias 27.3,
    # bias+res 27.1, +act 28.1 -- an erf GELU on 8 epilogue warps per SM (and
    # the pre-activation's second store) costs the FFN-up GEMM more than the
    # bias_act launch it replaces, so activations stay in bias_act
    fuse_epilogue = frozenset(x for x in os.environ.get("TALLY_FUSE_EPILOGUE", "bias,res").split(",") if x)

    def _init_common(self):
        import torch
        self.torch = torch
        self.sgd = SgdTable()
        self.program = []
        self.params = []

    def _finish(self, lr):
        self.sgd.build(self.device)
        self._add("sgd_update", K.sgd_update(self.sgd.dev_segs, self.sgd.dev_map, self.sgd.blocks, self.sgd.nbytes,
                                             lr, MOMENTUM))

    # ---- parameters -------------------------------------------------------------
    def _param(self, name, w32, bf16=True):
        torch = self.torch

        class Prm:
            pass
        p = Prm()
        p.name, p.w, p.v = name, w32.contiguous(), torch.zeros_like(w32)
        p.wb = p.w.bfloat16() if bf16 else None
        self.params.append((name, p.w))
        return p

    def _linear_w(self, name, w_out_in, b):
        """A linear layer from its [out, in] weight and bias."""
        lin = self._param(name + ".weight", w_out_in.contiguous().to(self.device))
        lin.b = self._param(name + ".bias", b.to(self.device).clone(), bf16=False)
        lin.out, lin.inp = lin.w.shape
        return lin

    def _ln_w(self, name, g, b):
        torch = self.torch

        class LN:
            pass
        ln = LN()
        ln.g = self._param(name + ".weight", g.to(self.device).clone(), bf16=False)
        ln.b = self._param(name + ".bias", b.to(self.device).clone(), bf16=False)
        ln.mean = torch.zeros(self.N, device=self.device)
        ln.rstd = torch.zeros(self.N, device=self.device)
        return ln

    def _buf(self, *shape, dtype=None):
        return self.torch.empty(*shape, dtype=dtype or self.torch.bfloat16, device=self.device)

    def _add(self, name, dk):
        self.program.append((name, dk))

    # ---- building blocks ------------------------------------------------------------
    def _colsum(self, name, g, dbeta, dgamma=None, x=None, mean=None, rstd=None, g2=None):
        P, C = g.shape
        rb = _rb_cols(P, C)
        nrb = (P + rb - 1) // rb
        part = self.torch.empty(2 * nrb * C, device=self.device)
        self._add(name, K.colstats(g, part, P, C, rb, dbeta, dgamma=dgamma, x=x, mean=mean, rstd=rstd, g2=g2))

    def _linear_fwd(self, name, lin, x, act=0, res=None, pre=None):
        fuse = "act" if act else "res" if res is not None else "bias"
        if fuse in self.fuse_epilogue:
            # y = act(x . W^T + b (+ res)) straight from the GEMM's TMA-store
            # epilogue (no split) or from the split-K reduce -- no bf16
            # intermediate, no bias_act launch
            M, N, Kd = self.N, lin.out, lin.inp
            pair, S = _pair_plan(M, N, Kd, self.pair_gemms)
            if S == 1 and (pair or N % 128 == 0):
                y = self._buf(M, N)
                self._add(name + ".gemm", K.gemm_ex(x, lin.wb, y, M, N, Kd, pair=pair, bias=lin.b.w, res=res,
                                                    pre=pre, act=act))
                return y
            if S > 1:
                y = self._buf(M, N)
                ws = self._ws(S * M * N).view(S * M, N)
                self._add(name + ".gemm", K.gemm_ex(x, lin.wb, ws, M, N, Kd, splits=S, pair=pair))
                self._add(name + ".reduce", K.splitk_reduce(ws.view(S, M, N), y, bias=lin.b.w, res=res, pre=pre,
                                                            act=act))
                return y
        u = self._buf(self.N, lin.out)
        self._gemm_ex_splitk(name + ".gemm", x, lin.wb, u, self.N, lin.out, lin.inp)
        y = self._buf(self.N, lin.out)
        self._add(name + ".bias", K.bias_act(u, y, lin.b.w, self.N, lin.out, act=act, res=res, pre=pre))
        return y

    def _add_tensors(self, name, a, b):
        """a + b (bf16, same shape): the residual branch of a post-LN gradient."""
        if not hasattr(self, "_zero_bias") or self._zero_bias.numel() < a.shape[1]:
            self._zero_bias = self.torch.zeros(max(a.shape[1], 4096), device=self.device)
        y = self._buf(*a.shape)
        self._add(name, K.bias_act(a, y, self._zero_bias, a.shape[0], a.shape[1], res=b))
        return y

    def _wgrad(self, name, p, dy, x):
        """dW[out, in] = dy^T . x, split-K fp32 partials -> sgd_update."""
        torch = self.torch
        M, Nn, Kd = dy.shape[1], x.shape[1], self.N
        pair, S = _pair_plan(M, Nn, Kd, self.pair_gemms)
        p.gpart = torch.empty(S, M, Nn, dtype=torch.float32, device=self.device)
        if S == 1:
            self._add(name + ".wgrad", K.gemm_ex(dy, x, p.gpart[0], M, Nn, Kd, a_mn=True, b_mn=True, pair=pair))
        else:
            self._add(name + ".wgrad", K.gemm_mn(dy, x, p.gpart, splits=S, pair=pair))
        self.sgd.add(p.w, p.v, p.gpart, S, M * Nn, WEIGHT_DECAY, p.wb, None, M, Nn)

    def _ws(self, numel):
        """Shared fp32 split-K workspace: the program's kernels run strictly in
        order, so one buffer serves every split-K GEMM; it grows by
        reallocation (earlier kernels keep their buffer alive)."""
        cur = getattr(self, "_wsbuf", None)
        if cur is None or cur.numel() < numel:
            self._wsbuf = cur = self.torch.empty(numel, dtype=self.torch.float32, device=self.device)
        return cur[:numel]

    def _gemm_ex_splitk(self, name, A, B, out, M, N, Kd, b_mn=False, res=None):
        """out (bf16) = A . B^T.  GEMMs with few, long output tiles (an LM-head
        dgrad with K = vocab; BERT-large's K = 4096 FFN GEMMs: 256 tiles of
        134 MFLOP) run split-K into an fp32 workspace + splitk_reduce, so their
        logical blocks are <= ~40 MFLOP (resnet._gemm_splits): short enough
        for a PTB configuration to meet the turnaround threshold, where the
        reference's fallback (least turnaround) would otherwise pick a 1/256
        slicing at 200x the latency.  ``res``: out = A . B^T + res (a
        residual-stream gradient), fused into the split-K reduce or the GEMM's
        TMA-store epilogue; returns False when it could not be fused."""
        pair, S = _pair_plan(M, N, Kd, self.pair_gemms)
        if S == 1:
            fuse = res is not None and "res" in self.fuse_epilogue and (pair or N % 128 == 0)
            self._add(name, K.gemm_ex(A, B, out, M, N, Kd, b_mn=b_mn, pair=pair, res=res if fuse else None))
            return fuse or res is None
        ws = self._ws(S * M * N).view(S * M, N)
        self._add(name, K.gemm_ex(A, B, ws, M, N, Kd, b_mn=b_mn, splits=S, pair=pair))
        fuse = res is not None and "res" in self.fuse_epilogue
        self._add(name + ".reduce", K.splitk_reduce(ws.view(S, M, N), out, res=res if fuse else None))
        return fuse or res is None

    def _linear_bwd(self, name, lin, dy, x, need_dx=True, res=None):
        """Bias and weight gradients of a linear layer; returns dx (+ ``res``,
        a residual-stream gradient added in the dgrad's epilogue when it can
        be fused, else by bias_act)."""
        lin.b.g = self.torch.zeros(lin.out, device=self.device)
        self._colsum(name + ".dbias", dy, lin.b.g)
        self.sgd.add(lin.b.w, lin.b.v, lin.b.g.view(1, -1), 1, lin.out, WEIGHT_DECAY)
        self._wgrad(name, lin, dy, x)
        if not need_dx:
            return None
        dx = self._buf(self.N, lin.inp)
        if not self._gemm_ex_splitk(name + ".dgrad", dy, lin.wb, dx, self.N, lin.inp, lin.out, b_mn=True, res=res):
            return self._add_tensors(name + ".residual_grad", dx, res)
        return dx

    def _ln_fwd(self, name, ln, x):
        y = self._buf(self.N, self.d)
        self._add(name, K.layernorm_fwd(x, y, ln.g.w, ln.b.w, ln.mean, ln.rstd, self.ln_eps))
        return y

    def _ln_bwd(self, name, ln, dy, x, g2=None):
        torch = self.torch
        ln.g.g = torch.zeros(self.d, device=self.device)
        ln.b.g = torch.zeros(self.d, device=self.device)
        self._colsum(name + ".dparams", dy, ln.b.g, dgamma=ln.g.g, x=x, mean=ln.mean, rstd=ln.rstd)
        self.sgd.add(ln.g.w, ln.g.v, ln.g.g.view(1, -1), 1, self.d, WEIGHT_DECAY)
        self.sgd.add(ln.b.w, ln.b.v, ln.b.g.view(1, -1), 1, self.d, WEIGHT_DECAY)
        dx = self._buf(self.N, self.d)
        self._add(name + ".bwd", K.layernorm_bwd(dy, x, ln.g.w, ln.mean, ln.rstd, dx, g2=g2))
        return dx

    # attention over (sequence, head) blocks of the fused QKV activation
    def _views(self, qkv):
        d = self.d
        return qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:]

    def _fused_attn(self):
        """S = Q.K^T + softmax (and dP + softmax backward) in one tcgen05 kernel
        whose scores never leave TMEM: all keys visible, T <= 512, head dim 64."""
        return self.fuse_attention and not self.causal and self.T % 128 == 0 and 128 <= self.T <= 512 \
            and self.D == 64

    def _attn_fwd(self, name, qkv, S, Pm):
        T, H, D = self.T, self.H, self.D
        q, k, v = self._views(qkv)
        z = dict(batches=self.B * H, hdiv=H)
        c1, c2 = (1, 2) if self.causal else (0, 0)   # causal tile / K-range rules (kernels.gemm_ex)
        if self._fused_attn():
            self._add(name + ".qk_softmax", K.attn_softmax(qkv, Pm, self.B, H, T, 1.0 / math.sqrt(D), d=self.d))
        else:
            self._add(name + ".qk", K.gemm_ex(q, k, S, T, T, D, a_off=((T, 0), (0, D)), b_off=((T, 0), (0, D)),
                                              c_off=((H * T, T), (0, 0)), causal=c1, **z))
            self._add(name + ".softmax", K.softmax_causal(S, Pm, T, 1.0 / math.sqrt(D), causal=self.causal))
        o = self._buf(self.N, self.d)
        self._add(name + ".pv", K.gemm_ex(Pm, v, o, T, D, T, b_mn=True, a_off=((H * T, T), (0, 0)),
                                          b_off=((T, 0), (0, D)), c_off=((T, 0), (0, D)), causal=c2, **z))
        return o

    def _attn_bwd(self, name, qkv, Pm, do, dP, dS):
        T, H, D = self.T, self.H, self.D
        q, k, v = self._views(qkv)
        z = dict(batches=self.B * H, hdiv=H)
        c1, c2, c3 = (1, 2, 3) if self.causal else (0, 0, 0)
        dqkv = self._buf(self.N, 3 * self.d)
        dq, dk_, dv = self._views(dqkv)
        if self._fused_attn():
            self._add(name + ".dp_softmax_bwd", K.attn_softmax_bwd(do, qkv, Pm, dS, self.B, H, T, 1.0 / math.sqrt(D),
                                                                   d=self.d))
        else:
            self._add(name + ".dp", K.gemm_ex(do, v, dP, T, T, D, a_off=((T, 0), (0, D)), b_off=((T, 0), (0, D)),
                                              c_off=((H * T, T), (0, 0)), causal=c1, **z))
            self._add(name + ".softmax_bwd", K.softmax_causal_bwd(Pm, dP, dS, T, 1.0 / math.sqrt(D),
                                                                  causal=self.causal))
        self._add(name + ".dq", K.gemm_ex(dS, k, dq, T, D, T, b_mn=True, a_off=((H * T, T), (0, 0)),
                                          b_off=((T, 0), (0, D)), c_off=((T, 0), (0, D)), causal=c2, **z))
        self._add(name + ".dk", K.gemm_ex(dS, q, dk_, T, D, T, a_mn=True, b_mn=True, a_off=((H * T, T), (0, 0)),
                                          b_off=((T, 0), (0, D)), c_off=((T, 0), (0, D)), causal=c3, **z))
        self._add(name + ".dv", K.gemm_ex(Pm, do, dv, T, D, T, a_mn=True, b_mn=True, a_off=((H * T, T), (0, 0)),
                                          b_off=((T, 0), (0, D)), c_off=((T, 0), (0, D)), causal=c3, **z))
        return dqkv

    # ---- running it -------------------------------------------------------------------
    def step_original(self, stream):
        launches = [dk.original(stream) for _, dk in self.program]
        for L in launches:
            L.wait()
        return launches[-1]

    def work_signature(self, name, dk):
        i = dk.info
        return f"{dk.kind}:{i.grid[0]}x{i.grid[1]}x{i.grid[2]}:{int(i.alg_bytes)}:{int(i.alg_flops)}"
