"""ResNet-50 workloads of config C2 (BASELINE.json configs[1]): bs=1 inference
as the high-priority task, bs=64 training as the best-effort task.

Best-effort training (``ResNet50Train``) is one training step written as a
fixed program of transformable device kernels -- every kernel of the step is
one of this package's sm_100a kinds in Original / Sliced / PTB shape, so the
scheduler can slice or preempt any of them (the paper transforms every kernel
of the best-effort job, §4).  Layout is NHWC bf16 ([P = N*H*W, C]
matrices); BN statistics and the optimizer run in fp32.

  conv (k x k or strided)  im2col_bf16 -> gemm (tcgen05)      [P, Kp] . W[Cout, Kp]^T
  conv (1 x 1, stride 1)   gemm directly on the activation
  batch-norm (training)    bn_stats -> bn_finalize -> bn_act (+ residual, ReLU)
  backward                 bn_stats(mode 1) -> bn_finalize -> bn_bwd;
                           dgrad gemm (+ col2im); wgrad = split-K gemm_mn reading
                           dY and the forward operand MN-major (no transposes)
  head                     avgpool -> gemm (fp32 logits) -> softmax_xent
  optimizer                sgd_update (momentum 0.9, weight decay 1e-4) over all
                           parameters, one launch

Weights are created from a torchvision ``resnet50()`` (random init -- no
checkpoints offline) so the parity tests can run the same step in PyTorch
fp32 and compare.  The input image is stored with 8 channels (3 real, 5 zero)
so every activation row is a whole number of 16-byte vectors.

High-priority inference (``ResNet50Infer``) runs unmodified, as the paper's
high-priority jobs do: the torchvision model in bf16 / channels-last captured
into a CUDA graph, launched as one exempt pipeline step at top priority.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

from . import kernels as K

STAGES = ((64, 256, 3, 1), (128, 512, 4, 2), (256, 1024, 6, 2), (512, 2048, 3, 2))
NUM_CLASSES = 1000
CLS_PAD = 1024
IN_CH = 8          # stored input channels (3 real + 5 zero)
MOMENTUM = 0.9
WEIGHT_DECAY = 1e-4
BN_EPS = 1e-5


def _rb(P, C, streams=1):
    """Rows per bn_stats logical block: ~128 KB of traffic per block (the
    per-block fixed cost -- partial write, fence, counter -- stays small) while
    a block still streams in a few microseconds; backward statistics read up
    to four streams.  (2x bigger backward blocks saved 0.14 ms per step but
    put bn_stats_bwd's preemption latency at ~58 us.)  Small tensors get
    shorter blocks so that at least ~2 waves of blocks (296) run in parallel."""
    base = (1024 if C < 128 else (512 if C < 256 else 256)) // streams
    cblocks = (C + 255) // 256
    return max(32, min(base, P * cblocks // 296 // 8 * 8))


def _FOLD_RB(C):
    """bn_fold rows per block: one load pass per block (the fold body covers
    256 / (min(C, 256) / 8) rows x 2 per pass: 64 rows at C = 64, 16 from 256)."""
    mode = os.environ.get("TALLY_BNFOLD_RB", "pass")   # experiment knob: "pass" or a fixed count
    if mode != "pass":
        return int(mode)
    return max(16, 64 * 64 // min(C, 256))


def _gemm_splits(M, N, Kdim):
    """Split-K factor for a GEMM: enough logical blocks of <= ~40 MFLOP each
    (~10-20 us on one SM, the preemption granularity) that the tuner finds a
    preemptible configuration under the turnaround threshold, without empty
    splits.  (20 MFLOP blocks cut the wgrad drain from ~19 to ~12 us but cost
    ~0.4 ms per step in split-K partial traffic.)"""
    bn = 128 if N % 128 == 0 else 64
    tiles = math.ceil(M / 128) * (N // bn)
    kb = math.ceil(Kdim / 64)
    flops = 2.0 * tiles * 128 * bn * Kdim
    want = max(tiles, math.ceil(flops / 40e6))
    # ... and, for half-empty tiles (M < 128: the weight gradients of
    # 64-channel layers, K = N*H*W), <= ~256 KB of operand bytes per block:
    # they are memory-bound, and 40 MFLOP blocks streamed ~620 KB each
    # (45-95 us: the C2 preemption tail).  sgd_update splits the resulting
    # many partials across thread groups.
    if M < 128:
        per_kb = 2 * (M + bn) * 64
        want = max(want, tiles * math.ceil(kb / max(2, 262144 // per_kb)))
    s = max(1, min(kb // 2, math.ceil(want / tiles)))
    return math.ceil(kb / math.ceil(kb / s))


def _pair_plan(M, N, Kdim, enabled=True):
    """(pair, splits) for a linear-layer GEMM.  CTA-pair tiles (256 x 256,
    ``*_x2`` kinds) when N % 256 == 0 and there are >= 32 of them (with the
    split below, enough blocks for the 74 SM pairs; measured: 64 -> 32 saves
    0.2 ms per BERT-large step, 0.5 ms per GPT-2 step); their logical blocks are capped at
    ~180 MFLOP (~8 us on a pair), so K = 3072 / 4096 GEMMs split three ways:
    at 270 MFLOP their PTB(148) Eq. 1 estimate sat at the 31.6 us threshold
    and measurement noise sometimes sent the tuner to its least-turnaround
    fallback (a 1/128 slicing).  Otherwise single-CTA tiles with
    ``resnet._gemm_splits``."""
    tiles = math.ceil(M / 256) * (N // 256) if N % 256 == 0 else 0
    if not enabled or tiles < int(os.environ.get("TALLY_PAIR_MIN_TILES", "32")):
        return False, _gemm_splits(M, N, Kdim)
    kb = math.ceil(Kdim / 64)
    s = max(1, min(kb // 2, math.ceil(2.0 * 256 * 256 * Kdim / 180e6)))
    return True, math.ceil(kb / math.ceil(kb / s))


@dataclass
class ConvSpec:
    name: str
    cin: int
    cout: int
    k: int
    stride: int
    pad: int
    h: int          # input spatial (square)
    w: int

    @property
    def oh(self):
        return (self.h + 2 * self.pad - self.k) // self.stride + 1

    @property
    def ow(self):
        return (self.w + 2 * self.pad - self.k) // self.stride + 1

    @property
    def kdim(self):
        return self.k * self.k * self.cin

    @property
    def kp(self):
        return (self.kdim + 63) // 64 * 64

    @property
    def direct(self):
        """1x1 stride-1 convolution: the activation is the GEMM operand."""
        return self.k == 1 and self.stride == 1


class SgdTable:
    """Packed ``nn::SgdSeg`` records + the logical-block map of sgd_update."""

    CHUNK = 1024     # max elements per sgd_update logical block

    def __init__(self):
        self.segs = []

    def add(self, w, v, grad, S, gstride, wd, wb=None, wt=None, rows=1, cols=1, zero_from=-1, wf=None, fk=0,
            fcin=0):
        """``zero_from`` >= 0: gradient slices [zero_from, S) are atomic
        accumulators, zeroed by sgd_update after it reads them.  ``wf``: the
        flipped bf16 copy of a k x k conv weight (``ResNet50Train._flip``)."""
        self.segs.append((w, v, grad, S, gstride, wd, wb, wt, rows, cols, zero_from, wf, fk, fcin))

    def build(self, device):
        import numpy as np
        import torch
        dt = np.dtype({"names": ["w", "v", "grad", "n", "gstride", "S", "wd", "wb", "wt", "rows", "cols", "chunk",
                                 "zero_from", "wf", "fk", "fcin"],
                       "formats": ["<u8", "<u8", "<u8", "<i8", "<i8", "<i4", "<f4", "<u8", "<u8", "<i4", "<i4", "<i4",
                                   "<i4", "<u8", "<i4", "<i4"],
                       "offsets": [0, 8, 16, 24, 32, 40, 44, 48, 56, 64, 68, 72, 76, 80, 88, 92], "itemsize": 96})
        rec = np.zeros(len(self.segs), dtype=dt)
        bmap = []
        nbytes = 0
        for i, (w, v, g, S, gs, wd, wb, wt, rows, cols, zf, wf, fk, fcin) in enumerate(self.segs):
            n = w.numel()
            if n % 4 or gs % 4:
                raise ValueError("sgd_update segments need sizes and gradient strides divisible by 4")
            # elements per logical block: ~32 KB of gradient partials read per
            # block (short blocks = short preemption latency), 1024 at most
            chunk = self.CHUNK
            while chunk > 64 and chunk * S * 4 > 32 * 1024:
                chunk //= 2
            rec[i] = (w.data_ptr(), v.data_ptr(), g.data_ptr(), n, gs, S, wd,
                      wb.data_ptr() if wb is not None else 0, wt.data_ptr() if wt is not None else 0,
                      rows, cols, chunk, zf, wf.data_ptr() if wf is not None else 0, fk, fcin)
            for c in range((n + chunk - 1) // chunk):
                bmap.append((i, c))
            nbytes += n * (4 * S + 16 + (2 if wb is not None else 0) + (2 if wt is not None else 0) +
                           (2 if wf is not None else 0))
        self.dev_segs = torch.from_numpy(rec.view(np.uint8).copy()).to(device)
        self.dev_map = torch.tensor(bmap, dtype=torch.int32, device=device)
        self.blocks = len(bmap)
        self.nbytes = nbytes
        self._keep = [s for s in self.segs]
        return self


class ResNet50Train:
    """One ResNet-50 training step (forward, backward, momentum SGD) as a
    fixed sequence of device kernels on preallocated HBM buffers.

    ``program`` lists ``(name, DeviceKernel)`` in execution order; ``data``
    holds the input batch [B, 224, 224, 8] bf16 and labels [B] int32 (refill
    them between steps); ``loss`` [B] fp32 holds per-sample losses after a
    step.  ``image`` may be smaller than 224 for tests (>= 32)."""

    # CTA-pair tcgen05 GEMMs where N % 256 == 0 and >= 32 pair tiles (_pair_plan)
    pair_gemms = os.environ.get("TALLY_RESNET_PAIR", "1") != "0"
    # implicit-GEMM convolutions (TMA im2col; see _implicit)
    implicit_conv = os.environ.get("TALLY_IMPLICIT_CONV", "1") != "0"
    implicit_dgrad = os.environ.get("TALLY_IMPLICIT_DGRAD", "1") != "0"
    # the stem through the narrow-channel implicit kinds: measured slower
    # (C2 step 10.21 -> 10.49 ms: one 16-byte gather per pixel and tap) than
    # im2col + GEMM, so off by default
    implicit_stem = os.environ.get("TALLY_IMPLICIT_STEM", "0") != "0"
    # batch-norm statistics fused into the producing GEMM / convolution
    # epilogue or split-K reduce (csrc/bnfuse.cuh): no bn_stats pass
    fuse_bn_stats = os.environ.get("TALLY_BN_FUSE", "1") != "0"
    # partial rows per 128 (one per tile, the epilogue warps combine through
    # shared memory) or per 32 output rows (one per warp, no exchange)
    bn_fuse_rows = int(os.environ.get("TALLY_BNFUSE_ROWS", "128"))

    def __init__(self, batch=64, image=224, lr=0.1, seed=0, device="cuda", model=None):
        import torch
        self.torch = torch
        self.B, self.image, self.lr, self.device = batch, image, lr, device
        self.program = []
        self.params = []          # (name, tensor) in torchvision naming, for parity
        self.sgd = SgdTable()
        self._scratch = {}
        self.acts = {}            # named forward activations (debugging / parity)
        self.block_grads = {}     # per bottleneck: upstream (g, g2) and produced (dx, dsc) gradients
        if model is None:
            import torchvision
            torch.manual_seed(seed)
            model = torchvision.models.resnet50(weights=None)
        self.ref_model = model
        sd = {k: v.detach().float() for k, v in model.state_dict().items()}
        dev = device
        B = batch
        self.x = torch.zeros(B, image, image, IN_CH, dtype=torch.bfloat16, device=dev)
        self.labels = torch.zeros(B, dtype=torch.int32, device=dev)
        self.loss = torch.zeros(B, dtype=torch.float32, device=dev)

        # ---- layers ---------------------------------------------------------
        h = image
        self.stem = self._conv(ConvSpec("conv1", IN_CH, 64, 7, 2, 3, h, h), sd["conv1.weight"])
        self.stem_bn = self._bn("bn1", 64, sd)
        h = self.stem.spec.oh
        self.pool_h = (h + 2 - 3) // 2 + 1
        blocks = []
        cin, hh = 64, self.pool_h
        for li, (width, cout, n, stride) in enumerate(STAGES):
            for bi in range(n):
                pre = f"layer{li + 1}.{bi}"
                s = stride if bi == 0 else 1
                blk = {"pre": pre, "cin": cin, "cout": cout, "width": width, "stride": s, "h": hh}
                blk["c1"] = self._conv(ConvSpec(pre + ".conv1", cin, width, 1, 1, 0, hh, hh), sd[pre + ".conv1.weight"])
                blk["b1"] = self._bn(pre + ".bn1", width, sd)
                blk["c2"] = self._conv(ConvSpec(pre + ".conv2", width, width, 3, s, 1, hh, hh), sd[pre + ".conv2.weight"])
                blk["b2"] = self._bn(pre + ".bn2", width, sd)
                ho = blk["c2"].spec.oh
                blk["c3"] = self._conv(ConvSpec(pre + ".conv3", width, cout, 1, 1, 0, ho, ho), sd[pre + ".conv3.weight"])
                blk["b3"] = self._bn(pre + ".bn3", cout, sd)
                if bi == 0:
                    blk["cd"] = self._conv(ConvSpec(pre + ".downsample.0", cin, cout, 1, s, 0, hh, hh),
                                           sd[pre + ".downsample.0.weight"])
                    blk["bd"] = self._bn(pre + ".downsample.1", cout, sd)
                blk["ho"] = ho
                blocks.append(blk)
                cin, hh = cout, ho
        self.blocks = blocks
        self.final_h = hh
        # classifier, classes padded to 1024 with zero rows
        fw = torch.zeros(CLS_PAD, 2048, device=dev)
        fw[:NUM_CLASSES] = sd["fc.weight"].to(dev)
        fb = torch.zeros(CLS_PAD, device=dev)
        fb[:NUM_CLASSES] = sd["fc.bias"].to(dev)
        self.fc_w, self.fc_v = fw, torch.zeros_like(fw)
        self.fc_wb = fw.bfloat16()
        self.fc_wt = fw.t().contiguous().bfloat16()
        self.fc_b, self.fc_bv = fb, torch.zeros_like(fb)
        self.params += [("fc.weight", fw), ("fc.bias", fb)]

        self._build_program()
        self.sgd.build(dev)
        self._add("sgd_update", K.sgd_update(self.sgd.dev_segs, self.sgd.dev_map, self.sgd.blocks,
                                              self.sgd.nbytes, self.lr, MOMENTUM))

    # ---- parameters ---------------------------------------------------------
    def _conv(self, spec, w_oihw):
        torch = self.torch
        dev = self.device
        cout, cin_real = w_oihw.shape[0], w_oihw.shape[1]
        w = torch.zeros(cout, spec.k, spec.k, spec.cin)
        w[..., :cin_real] = w_oihw.permute(0, 2, 3, 1)
        wm = torch.zeros(cout, spec.kp)
        wm[:, :spec.kdim] = w.reshape(cout, -1)
        wm = wm.to(dev)

        class Conv:
            pass
        c = Conv()
        c.spec, c.w, c.v = spec, wm, torch.zeros_like(wm)
        c.wb = wm.bfloat16()
        c.wt = wm.t().contiguous().bfloat16()
        c.wf = self._flip(wm, spec) if spec.cin % 64 == 0 and spec.k > 1 else None
        self.params.append((spec.name + ".weight", wm))
        return c

    @staticmethod
    def _flip(wm, spec):
        """[cout, (kh, kw, cin)] -> [cin, (k-1-kh, k-1-kw, cout)] bf16: the
        weight of dx as a stride-1 forward convolution of dy."""
        k, cin = spec.k, spec.cin
        w4 = wm[:, :spec.kdim].view(-1, k, k, cin)
        return w4.flip(1, 2).permute(3, 1, 2, 0).contiguous().view(cin, -1).bfloat16()

    def _bn(self, name, C, sd):
        torch = self.torch
        dev = self.device

        class BN:
            pass
        b = BN()
        b.name, b.C = name, C
        b.gamma = sd[name + ".weight"].to(dev).clone()
        b.beta = sd[name + ".bias"].to(dev).clone()
        b.vg, b.vb = torch.zeros_like(b.gamma), torch.zeros_like(b.beta)
        z = lambda: torch.zeros(C, device=dev)  # noqa: E731
        b.mean, b.invstd, b.dgamma, b.dbeta = z(), z(), z(), z()
        b.scale_shift = torch.zeros(2, C, device=dev)
        b.coef = torch.zeros(3, C, device=dev)
        self.params += [(name + ".weight", b.gamma), (name + ".bias", b.beta)]
        self.sgd.add(b.gamma, b.vg, b.dgamma, 1, C, WEIGHT_DECAY)
        self.sgd.add(b.beta, b.vb, b.dbeta, 1, C, WEIGHT_DECAY)
        return b

    # ---- buffers --------------------------------------------------------------
    def _buf(self, *shape, dtype=None):
        torch = self.torch
        return torch.empty(*shape, dtype=dtype or torch.bfloat16, device=self.device)

    def _scr(self, key, numel, dtype=None):
        """Shared scratch: kernels of the step run strictly in order on one
        stream, so transient operands (BN partials, dgrad columns, split-K
        workspaces) reuse one buffer per role, sized for the largest layer
        by _reserve_all."""
        cur = self._scratch.get(key)
        if cur is None or cur.numel() < numel or (dtype is not None and cur.dtype != dtype):
            raise RuntimeError(f"scratch {key!r} not reserved for {numel} elements")
        return cur[:numel]

    def _reserve(self, key, numel, dtype):
        cur = self._scratch.get(key)
        if cur is None or cur.numel() < numel:
            self._scratch[key] = self.torch.empty(numel, dtype=dtype, device=self.device)

    def _add(self, name, dk):
        self.program.append((name, dk))

    # ---- building blocks -----------------------------------------------------
    def _implicit(self, s):
        """k x k / strided convolution as an implicit GEMM (TMA im2col loads of
        the NHWC activation, no column matrix): every one but the stem (3
        channels padded to 8), which can go through the narrow-channel kinds
        (one 16-byte im2col load per filter tap; TALLY_IMPLICIT_STEM=1)."""
        return self.implicit_conv and not s.direct and (s.cin % 64 == 0 or (s.cin == IN_CH and self.implicit_stem))

    def _implicit_dgrad(self, s, conv):
        """Stride-1 "same" k x k convolutions: dx as an implicit-GEMM forward
        convolution of dy (cout % 64 == 0) with the flipped weight copy."""
        return self._implicit(s) and s.stride == 1 and 2 * s.pad == s.k - 1 and s.cout % 64 == 0 \
            and conv.wf is not None and self.implicit_dgrad

    def _conv_fwd(self, conv, x, bn=None):
        """x [P_in, Cin] -> (y [P_out, Cout], A operand [P_out, Kp]; for an
        implicit-GEMM convolution the input x itself, fused): with ``bn`` the
        producer also writes that batch norm's statistics (fused = True)."""
        s = conv.spec
        P = self.B * s.oh * s.ow
        y = self._buf(P, s.cout)
        if self._implicit(s):
            S = _gemm_splits(P, s.cout, s.kdim)
            geo = (self.B, s.h, s.w, s.cin, s.k, s.stride, s.pad)
            if S == 1:
                bno = self._bn_out(bn, P, self.bn_fuse_rows)
                self._add(s.name + ".gemm", K.conv_fprop(x, conv.wb, y, *geo, bn=bno))
                self._bn_fold(s.name + ".bnfold", bno, bn, P)
            else:
                ws = self._scr("splitk", S * P * s.cout, self.torch.float32).view(S, P, s.cout)
                self._add(s.name + ".gemm", K.conv_fprop(x, conv.wb, ws, *geo, splits=S))
                bno = self._reduce(s.name + ".gemm.reduce", ws, y, bn, P)
            return y, x, bno is not None
        if s.direct:
            A = x
        else:
            A = self._buf(P, s.kp)
            self._add(s.name + ".im2col", K.im2col(x, A, self.B, s.h, s.w, s.cin, s.k, s.k, s.stride, s.pad))
        fused = self._gemm(s.name + ".gemm", A, conv.wb, y, bn=bn)
        return y, A, fused

    def _bn_out(self, bn, P, rb):
        """The fused-statistics target of batch norm ``bn`` over P rows (None:
        not fused)."""
        if bn is None or not self.fuse_bn_stats:
            return None
        rows = K.BnStatsOut.gemm_rows(P, rb) if rb in (32, 128) else (P + rb - 1) // rb
        part = self._scr("part", 2 * rows * bn.C, self.torch.float32)
        return K.BnStatsOut(part, bn.gamma, bn.beta, bn.mean, bn.invstd, bn.scale_shift, BN_EPS, rb)

    def _bn_fold(self, name, bno, bn, P):
        """After a GEMM / convolution that wrote ``bno``'s partial rows: the
        fold into ``bn``'s statistics (bn_fold, 64 partial rows per block)."""
        if bno is None:
            return
        R = K.BnStatsOut.gemm_rows(P, bno.c.rb)
        rb = _FOLD_RB(bn.C)
        fpart = self._scr("bnfold", K.BnStatsOut.part_floats(R, bn.C, rb), self.torch.float32)
        fo = K.BnStatsOut(fpart, bn.gamma, bn.beta, bn.mean, bn.invstd, bn.scale_shift, BN_EPS, rb)
        self._add(name, K.bn_fold(bno.tensors[0], R, bn.C, P, fo))

    def _reduce(self, name, ws, out, bn, P):
        """Split-K sum into the bf16 ``out`` (with ``bn``'s statistics when
        fused); returns the statistics target or None."""
        bno = self._bn_out(bn, P, _rb(P, out.shape[1]))
        self._add(name, K.splitk_reduce(ws, out) if bno is None else K.splitk_reduce_bn(ws, out, bno))
        return bno

    def _gemm(self, name, A, B, out, bn=None):
        """out[M,N] (bf16) = A . B^T, split-K through an fp32 workspace when the
        GEMM has few, long output tiles (see _gemm_splits); with ``bn`` the
        batch-norm statistics of out are fused (returns whether they were)."""
        torch = self.torch
        M, Kd = A.shape
        N = B.shape[0]
        pair, S = _pair_plan(M, N, Kd, self.pair_gemms)
        if S == 1:
            bno = self._bn_out(bn, M, self.bn_fuse_rows)
            self._add(name, K.gemm(A, B, out, pair=pair, bn=bno))
            self._bn_fold(name + ".bnfold", bno, bn, M)
            return bno is not None
        ws = self._scr("splitk", S * M * N, torch.float32).view(S, M, N)
        self._add(name, K.gemm(A, B, ws, splits=S, pair=pair))
        return self._reduce(name + ".reduce", ws, out, bn, M) is not None

    def _bn_fwd(self, bn, y, P, relu, res=None, fused=False):
        torch = self.torch
        if not fused:
            rb = _rb(P, bn.C)
            nrb = (P + rb - 1) // rb
            part = self._scr("part", 2 * nrb * bn.C, torch.float32)
            self._add(bn.name + ".stats", K.bn_stats(y, part, P, bn.C, rb, bn.mean, bn.invstd, bn.gamma, bn.beta,
                                                     bn.scale_shift, BN_EPS))
        out = self._buf(P, bn.C)
        self._add(bn.name + ".act", K.bn_act(y, out, bn.scale_shift[0], bn.scale_shift[1], P, bn.C, relu, res))
        return out

    def _bn_bwd(self, bn, g, x, P, g2=None, mask=None, dz_out=None):
        torch = self.torch
        rb = _rb(P, bn.C, streams=4)
        nrb = (P + rb - 1) // rb
        part = self._scr("part", 2 * nrb * bn.C, torch.float32)
        dx = self._buf(P, bn.C)
        self._add(bn.name + ".bwd_stats", K.bn_stats_bwd(x, g, part, P, bn.C, rb, bn.mean, bn.invstd, bn.gamma,
                                                         bn.dgamma, bn.dbeta, bn.coef, g2=g2, y=mask))
        self._add(bn.name + ".bwd", K.bn_bwd(g, x, bn.coef[0], bn.coef[1], bn.coef[2], dx, P, bn.C, g2=g2, y=mask,
                                             dz_out=dz_out))
        return dx

    def _conv_bwd(self, conv, dy, A, need_dx=True):
        """dy [P_out, Cout]; A = the forward GEMM operand [P_out, Kp].
        Appends the weight gradient (split-K partials -> sgd_update) and
        returns dx [P_in, Cin] (or None)."""
        torch = self.torch
        s = conv.spec
        P = self.B * s.oh * s.ow
        # weight gradient: dW[Cout, Kp] = dy^T . A, both read MN-major as stored
        # (implicit GEMM: A = im2col(x) gathered by TMA im2col loads)
        if self._implicit(s):
            S = _gemm_splits(s.cout, s.kp, P)
            conv.gpart = torch.empty(S, s.cout, s.kp, dtype=torch.float32, device=self.device)
            self._add(s.name + ".wgrad", K.conv_wgrad(dy, A, conv.gpart, self.B, s.h, s.w, s.cin, s.k, s.stride,
                                                      s.pad, splits=S))
        else:
            pair, S = _pair_plan(s.cout, s.kp, P, self.pair_gemms)
            conv.gpart = torch.empty(S, s.cout, s.kp, dtype=torch.float32, device=self.device)
            self._add(s.name + ".wgrad", K.gemm_mn(dy, A, conv.gpart, splits=S, pair=pair))
        self.sgd.add(conv.w, conv.v, conv.gpart, S, s.cout * s.kp, WEIGHT_DECAY, conv.wb, conv.wt,
                     s.cout, s.kp, wf=conv.wf if self._implicit_dgrad(s, conv) else None, fk=s.k, fcin=s.cin)
        if not need_dx:
            return None
        # data gradient: dcol[P_out, Kp] = dy . W  (B operand = W^T [Kp, Cout])
        if s.direct:
            dx = self._buf(P, s.cin)
            self._gemm(s.name + ".dgrad", dy, conv.wt, dx)
            return dx
        if self._implicit_dgrad(s, conv):
            # dx = a stride-1 forward convolution of dy with the flipped weight
            # (padding k - 1 - pad): implicit GEMM, no column matrix, no col2im
            Pin = self.B * s.h * s.w
            dx = self._buf(Pin, s.cin)
            geo = (self.B, s.oh, s.ow, s.cout, s.k, 1, s.k - 1 - s.pad)
            S = _gemm_splits(Pin, s.cin, s.k * s.k * s.cout)
            if S == 1:
                self._add(s.name + ".dgrad", K.conv_fprop(dy, conv.wf, dx, *geo))
            else:
                ws = self._scr("splitk", S * Pin * s.cin, torch.float32).view(S, Pin, s.cin)
                self._add(s.name + ".dgrad", K.conv_fprop(dy, conv.wf, ws, *geo, splits=S))
                self._add(s.name + ".dgrad.reduce", K.splitk_reduce(ws, dx))
            return dx
        dcol = self._scr("dcol", P * s.kp).view(P, s.kp)
        self._gemm(s.name + ".dgrad", dy, conv.wt, dcol)
        dx = self._buf(self.B * s.h * s.w, s.cin)
        self._add(s.name + ".col2im", K.col2im(dcol, dx, self.B, s.h, s.w, s.cin, s.k, s.k, s.stride, s.pad))
        return dx

    def _all_convs(self):
        return [self.stem] + [b[k] for b in self.blocks for k in ("c1", "c2", "c3", "cd") if k in b]

    def _reserve_all(self):
        torch = self.torch
        convs = self._all_convs()
        part = dcol = splitk = 0
        for c in convs:
            s = c.spec
            P = self.B * s.oh * s.ow
            part = max(part, 2 * ((P + _rb(P, s.cout, 4) - 1) // _rb(P, s.cout, 4)) * s.cout,
                       2 * K.BnStatsOut.gemm_rows(P, 32) * s.cout)
            if not s.direct:
                dcol = max(dcol, P * s.kp)
            for (M, N, Kd) in ((P, s.cout, s.kp), (P, s.kp, s.cout)):     # forward, dgrad
                S = _pair_plan(M, N, Kd, self.pair_gemms)[1]
                if (M, N, Kd) == (P, s.cout, s.kp) and self._implicit(s):
                    S = _gemm_splits(M, N, Kd)   # (implicit-GEMM kinds are single-CTA)
                if (M, N, Kd) == (P, s.kp, s.cout) and self._implicit_dgrad(s, c):
                    Pin = self.B * s.h * s.w
                    S, M, N = _gemm_splits(Pin, s.cin, s.k * s.k * s.cout), Pin, s.cin
                if S > 1:
                    splitk = max(splitk, S * M * N)
        self._reserve("splitk", max(splitk, 8), torch.float32)
        self._reserve("part", part, torch.float32)
        self._reserve("bnfold", max(K.BnStatsOut.part_floats(K.BnStatsOut.gemm_rows(self.B * c.spec.oh * c.spec.ow, 32),
                                                             c.spec.cout, min(16, _FOLD_RB(c.spec.cout)))
                                    for c in convs), torch.float32)
        self._reserve("dcol", dcol, torch.bfloat16)

    # ---- the step ----------------------------------------------------------------
    def _build_program(self):
        torch = self.torch
        B = self.B
        self._reserve_all()
        # forward: stem
        st = self.stem.spec
        P1 = B * st.oh * st.ow
        y0, A0, f0 = self._conv_fwd(self.stem, self.x.view(B * self.image * self.image, IN_CH), self.stem_bn)
        a0 = self._bn_fwd(self.stem_bn, y0, P1, relu=True, fused=f0)
        P2 = B * self.pool_h * self.pool_h
        a1 = self._buf(P2, 64)
        arg = torch.empty(P2 * 64, dtype=torch.uint8, device=self.device)
        self._add("maxpool", K.maxpool_fwd(a0, a1, arg, B, st.oh, st.ow, 64))
        self.acts.update(stem_conv=y0, stem=a0, maxpool=a1)
        # forward: bottlenecks
        x = a1
        saved = []
        for blk in self.blocks:
            hh, ho = blk["h"], blk["ho"]
            Pin, Pout = B * hh * hh, B * ho * ho
            y1, A1, f1 = self._conv_fwd(blk["c1"], x, blk["b1"])
            o1 = self._bn_fwd(blk["b1"], y1, Pin, relu=True, fused=f1)
            y2, A2, f2 = self._conv_fwd(blk["c2"], o1, blk["b2"])
            o2 = self._bn_fwd(blk["b2"], y2, Pout, relu=True, fused=f2)
            y3, A3, f3 = self._conv_fwd(blk["c3"], o2, blk["b3"])
            if "cd" in blk:
                yd, Ad, fd = self._conv_fwd(blk["cd"], x, blk["bd"])
                sc = self._bn_fwd(blk["bd"], yd, Pout, relu=False, fused=fd)
            else:
                yd = Ad = None
                sc = x
            out = self._bn_fwd(blk["b3"], y3, Pout, relu=True, res=sc, fused=f3)
            self.acts[blk["pre"]] = out
            saved.append(dict(x=x, y1=y1, A1=A1, o1=o1, y2=y2, A2=A2, o2=o2, y3=y3, A3=A3, yd=yd, Ad=Ad,
                              out=out))
            x = out
        self.saved = saved
        # head
        hw = self.final_h * self.final_h
        feat = self._buf(B, 2048)
        self._add("avgpool", K.avgpool_fwd(x, feat, B, hw, 2048))
        logits = torch.empty(B, CLS_PAD, dtype=torch.float32, device=self.device)
        self._add("fc.gemm", K.gemm(feat, self.fc_wb, logits))
        dl = self._buf(B, CLS_PAD)
        dl32 = torch.empty(B, CLS_PAD, dtype=torch.float32, device=self.device)
        self._add("softmax_xent", K.softmax_xent(logits, self.fc_b, self.labels, self.loss, dl, dl32, NUM_CLASSES))
        self.logits = logits
        self.acts.update(feat=feat, logits=logits)
        # backward: head
        dfeat = self._buf(B, 2048)
        self._add("fc.dgrad", K.gemm(dl, self.fc_wt, dfeat))
        self.fc_g = torch.empty(1, CLS_PAD, 2048, dtype=torch.float32, device=self.device)
        self._add("fc.wgrad", K.gemm_mn(dl, feat, self.fc_g[0]))
        self.sgd.add(self.fc_w, self.fc_v, self.fc_g, 1, CLS_PAD * 2048, WEIGHT_DECAY, self.fc_wb, self.fc_wt,
                     CLS_PAD, 2048)
        self.sgd.add(self.fc_b, self.fc_bv, dl32, B, CLS_PAD, WEIGHT_DECAY)
        g = self._buf(B * hw, 2048)
        self._add("avgpool_bwd", K.avgpool_bwd(dfeat, g, B, hw, 2048))
        g2 = None
        # backward: bottlenecks
        for blk, sv in zip(reversed(self.blocks), reversed(saved)):
            hh, ho = blk["h"], blk["ho"]
            Pin, Pout = B * hh * hh, B * ho * ho
            dz = self._buf(Pout, blk["cout"])
            d3 = self._bn_bwd(blk["b3"], g, sv["y3"], Pout, g2=g2, mask=sv["out"], dz_out=dz)
            if "cd" in blk:
                dd = self._bn_bwd(blk["bd"], dz, sv["yd"], Pout)
                gsc = self._conv_bwd(blk["cd"], dd, sv["Ad"])
            else:
                gsc = dz
            dA3 = self._conv_bwd(blk["c3"], d3, sv["A3"])
            d2 = self._bn_bwd(blk["b2"], dA3, sv["y2"], Pout, mask=sv["o2"])
            dA2 = self._conv_bwd(blk["c2"], d2, sv["A2"])
            d1 = self._bn_bwd(blk["b1"], dA2, sv["y1"], Pin, mask=sv["o1"])
            dx = self._conv_bwd(blk["c1"], d1, sv["A1"])
            self.block_grads[blk["pre"]] = dict(g=g, g2=g2, dx=dx, dsc=gsc)
            g, g2 = dx, gsc
        # backward: stem
        da0 = self._buf(P1, 64)
        self._add("maxpool_bwd", K.maxpool_bwd(g, arg, da0, B, st.oh, st.ow, 64, dy2=g2))
        d0 = self._bn_bwd(self.stem_bn, da0, y0, P1, mask=a0)
        self._conv_bwd(self.stem, d0, A0, need_dx=False)

    # ---- running it ----------------------------------------------------------------
    @property
    def kernels(self):
        return [dk for _, dk in self.program]

    def step_original(self, stream):
        """Run the whole step untransformed on ``stream`` (the standalone
        baseline and the parity tests); returns the last launch."""
        launches = [dk.original(stream) for _, dk in self.program]
        for L in launches:
            L.wait()
        return launches[-1]

    def set_batch(self, images_nchw, labels):
        """images [B, 3, H, W] (any float dtype), labels [B] -> device buffers."""
        x = images_nchw.permute(0, 2, 3, 1).to(self.torch.bfloat16)
        self.x.zero_()
        self.x[..., :3].copy_(x)
        self.labels.copy_(labels.to(self.torch.int32))

    def conv_weight_oihw(self, conv):
        """A conv's fp32 master weight in torchvision layout (real input channels)."""
        s = conv.spec
        w = conv.w[:, :s.kdim].reshape(s.cout, s.k, s.k, s.cin).permute(0, 3, 1, 2)
        return w

    def work_signature(self, name, dk):
        """ProfileKey kernel name: the kind plus its launch geometry (each
        unique work configuration is profiled once)."""
        i = dk.info
        return f"{dk.kind}:{i.grid[0]}x{i.grid[1]}x{i.grid[2]}:{int(i.alg_bytes)}:{int(i.alg_flops)}"


class ResNet50Infer:
    """High-priority ResNet-50 inference request: the unmodified torchvision
    model (bf16, channels-last, cuDNN) captured into one CUDA graph.  The
    request pipeline is this single exempt step (``kernel``) -- high-priority
    kernels are launched as the application wrote them (§4.1)."""

    def __init__(self, batch=1, image=224, seed=1, device="cuda", persist_l2="nodes", warm_l2=True):
        import ctypes as C

        import torch
        import torchvision

        from . import _lib
        torch.manual_seed(seed)
        m = torchvision.models.resnet50(weights=None).eval()
        m = m.to(device=device, dtype=torch.bfloat16, memory_format=torch.channels_last)
        # all weights in one contiguous HBM range (the L2-persisting window)
        tensors = [t for t in list(m.parameters()) + list(m.buffers()) if t.is_floating_point()]
        total = sum(t.numel() for t in tensors)
        self.weights = torch.empty(total, dtype=torch.bfloat16, device=device)
        off = 0
        for t in tensors:
            n = t.numel()
            view = self.weights[off:off + n].view(t.shape)
            if t.dim() == 4:   # keep channels-last strides for the convolutions
                view = self.weights[off:off + n].view(t.shape[0], t.shape[2], t.shape[3], t.shape[1]).permute(0, 3, 1, 2)
            view.copy_(t)
            t.data = view
            off += n
        self.model = m
        self.inp = torch.randn(batch, 3, image, image, device=device, dtype=torch.bfloat16)
        self.inp = self.inp.contiguous(memory_format=torch.channels_last)
        side = torch.cuda.Stream()
        self.l2_window_bytes = 0
        if persist_l2 == "stream":
            # kernels captured from `side` carry the access-policy window: the
            # request's weights stay L2-resident next to a best-effort job
            win = C.c_longlong()
            _lib.check(_lib.lib.tally_l2_persist(C.c_void_p(side.cuda_stream), C.c_void_p(self.weights.data_ptr()),
                                                 self.weights.numel() * 2, 1.0, C.byref(win)), "l2 persist")
            self.l2_window_bytes = win.value
        side.wait_stream(torch.cuda.current_stream())
        with torch.no_grad():
            with torch.cuda.stream(side):
                for _ in range(3):
                    self.out = m(self.inp)
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            self.graph = torch.cuda.CUDAGraph(keep_graph=True)
            warm = torch.cuda.Stream() if warm_l2 else None
            with torch.cuda.graph(self.graph):
                if warm is not None:
                    # fork: an L2 warm-up of the weights runs next to the first
                    # layers, so a request that follows best-effort traffic
                    # finds the later layers' weights in L2 again
                    warm.wait_stream(torch.cuda.current_stream())
                    with torch.cuda.stream(warm):
                        _lib.check(_lib.lib.tally_l2_prefetch(C.c_void_p(warm.cuda_stream),
                                                              C.c_void_p(self.weights.data_ptr()),
                                                              self.weights.numel() * 2), "l2 prefetch")
                self.out = m(self.inp)
                if warm is not None:
                    torch.cuda.current_stream().wait_stream(warm)
        torch.cuda.synchronize()
        if persist_l2 == "nodes":
            # every kernel node of the request graph keeps the weights L2-persisting
            nodes = C.c_int()
            _lib.check(_lib.lib.tally_graph_l2_persist(C.c_void_p(self.graph.raw_cuda_graph()),
                                                       C.c_void_p(self.weights.data_ptr()),
                                                       self.weights.numel() * 2, 1.0, C.byref(nodes)),
                       "graph l2 persist")
            self.l2_window_bytes = self.weights.numel() * 2
            self.l2_nodes = nodes.value
        self.graph.instantiate()
        self.kernel = K.cuda_graph(self.graph)

    def reference(self):
        """Eager forward of the same model on the same input (parity)."""
        import torch
        with torch.no_grad():
            return self.model(self.inp)
