"""Registered device kernels and their three launch shapes.

A :class:`DeviceKernel` is a built-in sm_100a kernel bound to device buffers
(``tally_kernel_create``): it has a *logical grid* -- the untransformed launch
-- and can be launched as

* ``original()``                       the untransformed kernel,
* ``sliced(offset, count)``            a contiguous range of logical blocks
                                       (ref transforms.py:155-197),
* ``ptb(workers, start_count, ...)``   persistent preemptible workers resuming
                                       from a persisted task counter
                                       (ref transforms.py:291-448).

Buffers are torch tensors owned by the caller; the kernel keeps a reference
for its lifetime.
"""

from __future__ import annotations

import ctypes as C

_ctypes = C   # (gemm() names its output C)
from dataclasses import dataclass

from . import _lib
from .device import B200Device, KernelCostModel, DEFAULT_LAUNCH_OVERHEAD_NS


def _ptr(t):
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        if not t.is_cuda:
            raise ValueError("device kernels need CUDA tensors")
        if not t.is_contiguous():
            raise ValueError("device kernels need contiguous tensors")
        return t.data_ptr()
    return int(t)


class Stream:
    """A CUDA stream at the greatest (HIGH) or least (BEST_EFFORT) priority."""

    def __init__(self, high_priority: bool):
        B200Device.get()
        sid = C.c_int()
        _lib.check(_lib.lib.tally_stream_create(_lib.HIGH_CLASS if high_priority
                                                else _lib.BEST_EFFORT_CLASS, C.byref(sid)),
                   "stream")
        self.id = sid.value

    def synchronize(self):
        _lib.check(_lib.lib.tally_stream_sync(self.id), "stream sync")

    def handle(self) -> int:
        """The cudaStream_t (e.g. for torch.cuda.ExternalStream)."""
        h = C.c_void_p()
        _lib.check(_lib.lib.tally_stream_handle(self.id, C.byref(h)), "stream handle")
        return h.value or 0

    def close(self):
        if self.id >= 0:
            _lib.lib.tally_stream_destroy(self.id)
            self.id = -1


@dataclass
class LaunchState:
    done: bool
    parked: bool
    preempted: bool
    task_counter: int
    claims: int
    gt_first_start: int
    gt_first_stop: int
    gt_last_exit: int
    host_submit_ns: int
    host_preempt_ns: int
    gt_last_busy_exit: int = 0   # last exit of a worker that ran a block (late starters excluded)


def _state(s: _lib.c_launch_state) -> LaunchState:
    return LaunchState(bool(s.done), bool(s.parked), bool(s.preempted), s.task_counter, s.claims,
                       s.gt_first_start, s.gt_first_stop, s.gt_last_exit, s.host_submit_ns,
                       s.host_preempt_ns, s.gt_last_busy_exit)


class Launch:
    """One in-flight launch (a KernelHandle on the real device)."""

    def __init__(self, lid: int, shape: int):
        self.id = lid
        self.shape = shape
        self._final = None

    def query(self) -> LaunchState:
        if self._final is not None:
            return self._final
        s = _lib.c_launch_state()
        _lib.check(_lib.lib.tally_launch_query(self.id, C.byref(s)), "launch query")
        st = _state(s)
        if st.done or st.parked:
            self._finish(st)
        return st

    def wait(self) -> LaunchState:
        if self._final is not None:
            return self._final
        s = _lib.c_launch_state()
        _lib.check(_lib.lib.tally_launch_wait(self.id, C.byref(s)), "launch wait")
        st = _state(s)
        self._finish(st)
        return st

    def _finish(self, st):
        self._final = st
        self._elapsed = None
        v = C.c_longlong()
        if _lib.lib.tally_launch_elapsed_ns(self.id, C.byref(v)) == 0:
            self._elapsed = v.value
        _lib.lib.tally_launch_release(self.id)

    @property
    def elapsed_ns(self):
        """Device time between the launch's bracketing events (timed launches)."""
        if self._final is None:
            self.wait()
        return self._elapsed

    def preempt(self):
        _lib.check(_lib.lib.tally_preempt(self.id), "preempt")


@dataclass(frozen=True)
class KernelInfo:
    grid: tuple
    total_blocks: int
    threads_per_block: int
    smem_bytes: int
    occupancy_ptb: int
    occupancy_original: int
    alg_bytes: float
    alg_flops: float
    preempt_units: int = 1
    cluster: int = 1      # CTAs per logical block (CTA-pair GEMMs: 2)


class DeviceKernel:
    """A built-in kernel kind bound to arguments (``tally_kernel_create``)."""

    def __init__(self, kind: str, ptrs=(), ints=(), floats=(), keep=()):
        B200Device.get()
        a = _lib.c_kernel_args()
        for i, p in enumerate(ptrs):
            a.ptr[i] = _ptr(p)
        for i, v in enumerate(ints):
            a.i[i] = int(v)
        for i, v in enumerate(floats):
            a.f[i] = float(v)
        kid = C.c_int()
        _lib.check(_lib.lib.tally_kernel_create(kind.encode(), C.byref(a), C.byref(kid)), kind)
        self.kind = kind
        self.id = kid.value
        self._keep = tuple(keep) + tuple(p for p in ptrs if hasattr(p, "data_ptr"))
        ki = _lib.c_kernel_info()
        _lib.check(_lib.lib.tally_kernel_info_get(self.id, C.byref(ki)), "kernel info")
        self.info = KernelInfo((ki.grid_x, ki.grid_y, ki.grid_z), ki.total_blocks,
                               ki.threads_per_block, ki.smem_bytes, ki.occupancy_ptb,
                               ki.occupancy_original, ki.alg_bytes, ki.alg_flops,
                               max(1, ki.preempt_units), max(1, ki.cluster))

    @property
    def total_blocks(self) -> int:
        return self.info.total_blocks

    def full_workers(self, sms: int = 148) -> int:
        """PTB workers (CTAs) for a full-occupancy launch: every resident slot,
        at most one per logical block, a multiple of the cluster size."""
        cl = max(1, self.info.cluster)
        w = min(self.total_blocks * cl, sms * max(1, self.info.occupancy_ptb))
        return max(cl, w // cl * cl)

    def _launch(self, stream: Stream, desc: _lib.c_launch_desc) -> Launch:
        lid = C.c_int()
        _lib.check(_lib.lib.tally_launch(self.id, stream.id, C.byref(desc), C.byref(lid)),
                   f"{self.kind} launch")
        return Launch(lid.value, desc.shape)

    def original(self, stream: Stream, exec_count=None, timed=False, block_log=None) -> Launch:
        """``block_log``: optional uint64/int64 CUDA tensor [total_blocks, 3]
        receiving per logical block (start, end, smid) on the device clock."""
        d = _lib.c_launch_desc(shape=_lib.SHAPE_ORIGINAL, preempt_at=-1,
                               exec_count=_ptr(exec_count), timed=int(timed), block_log=_ptr(block_log))
        return self._launch(stream, d)

    def sliced(self, stream: Stream, offset: int, count: int, exec_count=None,
               timed=False, block_log=None) -> Launch:
        """Logical blocks [offset, offset + count) of the x-fastest order."""
        d = _lib.c_launch_desc(shape=_lib.SHAPE_SLICED, linear=1, linear_offset=offset,
                               count=count, preempt_at=-1, exec_count=_ptr(exec_count),
                               timed=int(timed), block_log=_ptr(block_log))
        return self._launch(stream, d)

    def sliced_rect(self, stream: Stream, offset, sub_grid, exec_count=None) -> Launch:
        """Rectangular sub-grid at a 3-D block offset (ref transforms.py:92-133)."""
        d = _lib.c_launch_desc(shape=_lib.SHAPE_SLICED, linear=0, off_x=offset[0],
                               off_y=offset[1], off_z=offset[2], sub_x=sub_grid[0],
                               sub_y=sub_grid[1], sub_z=sub_grid[2], preempt_at=-1,
                               exec_count=_ptr(exec_count))
        return self._launch(stream, d)

    def ptb(self, stream: Stream, workers: int, start_count: int = 0, preempt_at=None,
            exec_count=None, timed=False, worker_log=None, chain=False, block_log=None) -> Launch:
        """``worker_log``: optional int64 CUDA tensor [workers, 4] receiving per
        worker ``(smid << 32 | blocks done, t_entry, t_exit, stopped)`` on the
        device %globaltimer clock.  ``chain``: park on the stream's shared
        chain word (preempting this launch parks every chain launch queued
        behind it on the stream)."""
        d = _lib.c_launch_desc(shape=_lib.SHAPE_PTB, workers=workers, start_count=start_count,
                               preempt_at=-1 if preempt_at is None else preempt_at,
                               exec_count=_ptr(exec_count), worker_log=_ptr(worker_log),
                               timed=int(timed), chain=int(chain), block_log=_ptr(block_log))
        return self._launch(stream, d)

    def cost(self, block_duration_ns: int = 0, launch_overhead_ns: int = DEFAULT_LAUNCH_OVERHEAD_NS,
             ptb_iteration_overhead_ns: int = 0) -> KernelCostModel:
        """The KernelCostModel this kernel registers with (durations are
        informational on the B200; the profiler measures the real ones)."""
        return KernelCostModel(block_duration_ns, launch_overhead_ns, ptb_iteration_overhead_ns,
                               self.info.threads_per_block, self.info.total_blocks)

    def close(self):
        if self.id >= 0:
            _lib.lib.tally_kernel_destroy(self.id)
            self.id = -1
            self._keep = ()


# -- constructors for the built-in kinds ------------------------------------
def vecadd_i64(mem, a_base: int, b_base: int, out_base: int, n: int,
               elems_per_block: int = 1) -> DeviceKernel:
    """IR vecadd over an int64 word image ``[a | b | out]`` (ref tests/test_ir.py:165-172)."""
    return DeviceKernel("vecadd_i64", (mem,), (a_base, b_base, out_base, n, elems_per_block))


def vecadd_f32(a, b, c) -> DeviceKernel:
    """c = a + b; 4096 elements per logical block."""
    return DeviceKernel("vecadd_f32", (a, b, c), (a.numel(),))


def rowsum_f32(x, out) -> DeviceKernel:
    """out[r] = sum(x[r, :]); 8 rows per logical block."""
    rows, cols = x.shape
    return DeviceKernel("rowsum_f32", (x, out), (rows, cols))


def kind_names():
    n = _lib.lib.tally_kernel_kind_count()
    return [_lib.lib.tally_kernel_kind_name(i).decode() for i in range(n)]


class Sgemm3xTf32:
    """C[M,N] = A[M,K] . B[N,K]^T in fp32 accuracy on the tensor cores.

    Three device kernels: ``split_a`` / ``split_b`` (``split_tf32``: x -> tf32
    hi + fp32 remainder, HBM bound) and ``gemm`` (``sgemm_tf32x3``: tcgen05
    kind::tf32, Ahi.Bhi + Ahi.Blo + Alo.Bhi in fp32 TMEM).  ``pipeline`` lists
    them in order -- one BE training "step" of the SGEMM workload.
    """

    def __init__(self, A, B, C, chunk_preempt: bool = True, tile_n: int = 128):
        import torch
        M, K = A.shape
        N, K2 = B.shape
        if K != K2 or tuple(C.shape) != (M, N):
            raise ValueError("sgemm_tf32x3: shapes must be A[M,K], B[N,K], C[M,N]")
        if A.dtype != torch.float32 or B.dtype != torch.float32 or C.dtype != torch.float32:
            raise ValueError("sgemm_tf32x3: fp32 operands")
        self.a_hi, self.a_lo = torch.empty_like(A), torch.empty_like(A)
        self.b_hi, self.b_lo = torch.empty_like(B), torch.empty_like(B)
        self.split_a = DeviceKernel("split_tf32", (A, self.a_hi, self.a_lo), (A.numel(),))
        self.split_b = DeviceKernel("split_tf32", (B, self.b_hi, self.b_lo), (B.numel(),))
        kind = {128: "sgemm_tf32x3", 64: "sgemm_tf32x3_n64"}[tile_n]
        self.gemm = DeviceKernel(kind, (self.a_hi, self.a_lo, self.b_hi, self.b_lo, C),
                                 (M, N, K, 0 if chunk_preempt else 1))
        self.pipeline = (self.split_a, self.split_b, self.gemm)

    def prepare(self, stream: Stream):
        """Run the two splits (Original shape) and wait."""
        self.split_a.original(stream).wait()
        self.split_b.original(stream).wait()

    def close(self):
        for k in self.pipeline:
            k.close()


def sgemm_tf32x3(A, B, C, chunk_preempt: bool = True, tile_n: int = 128) -> Sgemm3xTf32:
    """``chunk_preempt``: PTB workers yield at every 256-deep K chunk, saving
    the fp32 partial tile (default); False = block (tile) granularity only."""
    return Sgemm3xTf32(A, B, C, chunk_preempt, tile_n)


def gemm_bf16(A, B, C) -> DeviceKernel:
    """C[M,N] (bf16) = A[M,K] . B[N,K]^T, bf16 operands, fp32 accumulation."""
    M, K = A.shape
    N, K2 = B.shape
    if K != K2 or tuple(C.shape) != (M, N):
        raise ValueError("gemm_bf16: shapes must be A[M,K], B[N,K], C[M,N]")
    return DeviceKernel("gemm_bf16", (A, B, C), (M, N, K))


def memcpy(dst, src, nbytes: int | None = None) -> DeviceKernel:
    """A host<->device copy step of a request pipeline (``cudaMemcpyAsync`` on
    the launch stream).  Copies are exempt from transformation -- register
    them with ``KernelWork(..., exempt=True)``; only ``original()`` launches."""
    nb = nbytes if nbytes is not None else src.numel() * src.element_size()
    if dst.numel() * dst.element_size() < nb:
        raise ValueError("memcpy: destination too small")
    return DeviceKernel("memcpy", (dst.data_ptr(), src.data_ptr()), (nb,), keep=(dst, src))


def cuda_graph(graph) -> DeviceKernel:
    """An unmodified program -- a captured ``torch.cuda.CUDAGraph`` (e.g. a
    model's inference forward) -- as one exempt pipeline step, launched with
    ``cudaGraphLaunch`` on the scheduler's stream of its priority."""
    exec_handle = graph.raw_cuda_graph_exec() if hasattr(graph, "raw_cuda_graph_exec") else int(graph)
    return DeviceKernel("cuda_graph", (int(exec_handle),), (), keep=(graph,))


EWISE_OPS = {"add": 0, "mul": 1, "relu": 2, "gelu": 3, "gelu_tanh": 4, "silu": 5}


def ewise(op: str, a, b, out, alpha: float = 1.0) -> DeviceKernel:
    """out = op(a[, b]) elementwise over contiguous fp32 or bf16 tensors of the
    same shape (``add``: a + alpha * b; ``mul``; unary ``relu``, ``gelu``
    (erf), ``gelu_tanh``, ``silu``): fp32 arithmetic, one rounding to the
    output type.  ``out`` may alias ``a`` (in-place ops)."""
    import torch
    bf16 = a.dtype == torch.bfloat16
    return DeviceKernel("ewise", (a, b, out), (a.numel(), EWISE_OPS[op], int(bf16)), (alpha,))


def spin(total_blocks: int, threads_per_block: int, block_duration_ns: int) -> DeviceKernel:
    """A cost-model kernel (ref ``KernelCostModel``): ``total_blocks`` logical
    blocks of ``threads_per_block`` threads, each holding its slot for
    ``block_duration_ns`` -- the reference's abstract workloads on the GPU."""
    return DeviceKernel("spin", (), (total_blocks, threads_per_block, block_duration_ns))


# -- best-effort training kinds (config C2, kernels_nn.cu) ---------------------
def _pack_conv(kh, kw, stride, pad):
    return kh | (kw << 8) | (stride << 16) | (pad << 24)


def _pair_suffix(pair: bool, N: int) -> str:
    if not pair:
        return ""
    if N % 256:
        raise ValueError("CTA-pair GEMMs (256 x 256 tiles) need N % 256 == 0")
    return "_x2"


class BnStatsOut:
    """Where a producer kernel writes the training batch-norm statistics of
    its bf16 output [P, C] (``tally_bn_stats``): ``part`` fp32 scratch, the
    layer's gamma / beta, and the outputs mean, invstd and scale_shift [2, C]
    -- what ``bn_stats`` computes from the stored tensor, fused into the
    GEMM / convolution epilogue or ``splitk_reduce_bn``."""

    def __init__(self, part, gamma, beta, mean, invstd, scale_shift, eps=1e-5, rb=0):
        self.tensors = (part, gamma, beta, mean, invstd, scale_shift)
        s = _lib.c_bn_stats()
        s.part, s.gamma, s.beta, s.mean, s.invstd, s.scale_shift = (t.data_ptr() for t in self.tensors)
        s.eps, s.rb = float(eps), int(rb)
        self.c = s

    @staticmethod
    def part_floats(P, C, rb=128):
        """fp32 scratch floats of a fold over P rows, rb per block."""
        return 2 * ((P + rb - 1) // rb) * C

    @staticmethod
    def gemm_rows(P, rb=128):
        """Partial rows a GEMM / conv_fprop epilogue writes for P output rows:
        one per 128-row tile, or (rb = 32) one per epilogue warp."""
        return (P + 127) // 128 * (4 if rb == 32 else 1)


def gemm(A, B, C, splits: int = 1, pair: bool = False, bn: "BnStatsOut | None" = None) -> DeviceKernel:
    """C[M,N] = A[M,K] . B[N,K]^T on tcgen05 (bf16 operands, fp32 accumulation).

    The kind follows the operands: N % 128 == 0 -> 128-wide tiles, else
    64-wide; C bf16 or fp32.  ``splits`` > 1 (fp32 C of shape [splits, M, N])
    is split-K: logical block = (split, tile), each split writing its own
    fp32 partial (summed later by ``sgd_update``).  ``pair``: a CTA pair
    (cluster of two SMs, ``tcgen05.mma.cta_group::2``) per 256 x 256 tile --
    one logical block per pair, PTB workers in CTAs (a multiple of 2)."""
    import torch
    M, K = A.shape
    N, K2 = B.shape
    if K != K2:
        raise ValueError("gemm: A[M,K], B[N,K] need the same K")
    out_f32 = C.dtype == torch.float32
    if tuple(C.shape[-2:]) != (M, N) or (splits > 1 and (not out_f32 or C.numel() != splits * M * N)):
        raise ValueError("gemm: C must be [M,N] (or [splits,M,N] fp32 for split-K)")
    kind = "gemm_bf16" + ("f32" if out_f32 else "") + (_pair_suffix(True, N) if pair else
                                                       "" if N % 128 == 0 else "_n64")
    if bn is None:
        return DeviceKernel(kind, (A, B, C), (M, N, K, 0, splits))
    return DeviceKernel(kind, (A, B, C, None, None, None, None, _ctypes.addressof(bn.c)), (M, N, K, 0, splits),
                        keep=(bn, bn.tensors))


def gemm_ex(A, B, Cout, M, N, K, a_mn=False, b_mn=False, splits=1, batches=1, hdiv=1,
            a_off=((0, 0), (0, 0)), b_off=((0, 0), (0, 0)), c_off=((0, 0), (0, 0)), causal=0,
            pair=False, bias=None, res=None, pre=None, act=0) -> DeviceKernel:
    """General bf16 GEMM on tcgen05: per batch, C[M,N] = A . B^T with A
    K-major (A[M,K] row-major) or MN-major (stored as A^T [K,M]), likewise B
    ([N,K] or [K,N]).  ``A``, ``B``, ``Cout`` are 2-D row-major views (any
    column offset and row pitch, e.g. one head's columns of a fused QKV
    activation).  Batch z = (zb, zh) = (z // hdiv, z % hdiv) moves each
    operand's (row, col) origin by off[0] * zb + off[1] * zh, with
    ``a_off = ((row_per_zb, row_per_zh), (col_per_zb, col_per_zh))``.
    bf16 or fp32 output; fp32 allows split-K.  ``causal`` (causal attention,
    T x T per batch, T % 128 == 0): 1 = S = Q.K^T / dP = dO.V^T, tiles wholly
    above the diagonal skipped (left unwritten); 2 = P.V / dS.K, K limited to
    keys <= the tile's last query; 3 = dS^T.Q / P^T.dO, K from the tile's
    first key.  ``pair``: CTA-pair kind (256 x 256 tiles, N % 256 == 0; not
    causal; ``_mn`` only with fp32 output).  ``bias`` (fp32 [N]) fuses the
    linear-layer epilogue into a plain bf16 GEMM: Cout = act(A.B^T + bias
    (+ res)), ``pre`` receiving the pre-activation (``bias_act`` semantics on
    the fp32 accumulator; res / pre share Cout's row pitch)."""
    import torch
    kinds = {(False, False): "", (True, True): "_mn", (False, True): "_kmn"}
    if (a_mn, b_mn) not in kinds:
        raise ValueError("gemm_ex: an MN-major A needs an MN-major B")
    for t in (A, B, Cout):
        if t.dim() != 2 or t.stride(1) != 1:
            raise ValueError("gemm_ex: operands must be 2-D row-major views (unit column stride)")
    out = "f32" if Cout.dtype == torch.float32 else ""
    kind = "gemm_bf16" + out + kinds[(a_mn, b_mn)] + (_pair_suffix(True, N) if pair else
                                                      "" if N % 128 == 0 else "_n64")
    lay = _lib.c_gemm_layout()
    lay.a_rows, lay.a_cols, lay.a_ld = A.shape[0], A.shape[1], A.stride(0)
    lay.b_rows, lay.b_cols, lay.b_ld = B.shape[0], B.shape[1], B.stride(0)
    lay.ldc = Cout.stride(0)
    lay.batches, lay.hdiv = batches, hdiv
    for name, (r, c) in (("a", a_off), ("b", b_off), ("c", c_off)):
        getattr(lay, name + "_row_off")[0], getattr(lay, name + "_row_off")[1] = r
        getattr(lay, name + "_col_off")[0], getattr(lay, name + "_col_off")[1] = c
    ep = tuple(t for t in (bias, res, pre) if t is not None)
    return DeviceKernel(kind, (A.data_ptr(), B.data_ptr(), Cout.data_ptr(), C.addressof(lay),
                               _ptr(bias), _ptr(res), _ptr(pre)),
                        (M, N, K, 0, splits, causal, act), keep=(A, B, Cout, lay) + ep)


def attn_softmax(qkv, P, B, H, T, scale, d=None) -> DeviceKernel:
    """Fused S = Q.K^T and P = softmax(scale * S) for every (sequence, head),
    all keys visible (T in 128..512, head dim 64): Q / K are the head slices
    of the fused QKV activation [B*T, 3d]; P is [B*H*T, T] bf16.  The fp32
    scores stay in TMEM."""
    d = d if d is not None else qkv.shape[1] // 3
    ld = qkv.stride(0)
    return DeviceKernel("attn_softmax", (qkv, qkv, P, None), (B, H, T, ld, ld, 0, d), (scale,))


def attn_softmax_bwd(dO, qkv, P, dS, B, H, T, scale, d=None) -> DeviceKernel:
    """Fused dP = dO.V^T and dS = P * (dP - rowsum(P * dP)) * scale (the
    softmax backward of ``attn_softmax``); dO [B*T, d], V the third head
    slice of the fused QKV activation, P / dS [B*H*T, T] bf16."""
    d = d if d is not None else qkv.shape[1] // 3
    return DeviceKernel("attn_softmax_bwd", (dO, qkv, dS, P), (B, H, T, dO.stride(0), qkv.stride(0), 0, 2 * d),
                        (scale,))


def gemm_mn(At, Bt, C, splits: int = 1, pair: bool = False) -> DeviceKernel:
    """C[M,N] (fp32) = At[K,M]^T . Bt[K,N] with both operands MN-major (as
    stored: M / N contiguous) -- the weight gradient dW = dY^T . X of a
    convolution straight from the NHWC activations.  Split-K as ``gemm``."""
    import torch
    K, M = At.shape
    K2, N = Bt.shape
    if K != K2:
        raise ValueError("gemm_mn: At[K,M], Bt[K,N] need the same K")
    if C.dtype != torch.float32 or tuple(C.shape[-2:]) != (M, N) or C.numel() != splits * M * N:
        raise ValueError("gemm_mn: C must be fp32 [M,N] (or [splits,M,N])")
    kind = "gemm_bf16f32_mn" + (_pair_suffix(True, N) if pair else "" if N % 128 == 0 else "_n64")
    return DeviceKernel(kind, (At, Bt, C), (M, N, K, 0, splits))


def _conv_geom(n, h, w, c, k, stride, pad):
    g = _lib.c_conv_geometry()
    g.n, g.h, g.w, g.c, g.k, g.stride, g.pad = n, h, w, c, k, stride, pad
    return g


def conv_fprop(x, Wt, out, n, h, w, c, k, stride, pad, splits: int = 1,
               bn: "BnStatsOut | None" = None) -> DeviceKernel:
    """Implicit-GEMM convolution: out[P, cout] = im2col(x) . Wt^T with the
    im2col operand gathered by TMA im2col loads straight from the NHWC input
    x [n, h, w, c] (c % 64 == 0) -- no column matrix.  Wt [cout, k*k*c] in
    (kh, kw, c) order.  bf16 out, or fp32 split-K partials [splits, P, cout]."""
    import torch
    cout = Wt.shape[0]
    ho = (h + 2 * pad - k) // stride + 1
    wo = (w + 2 * pad - k) // stride + 1
    P = n * ho * wo
    if c == 8:
        # 8-channel input (the ResNet stem): a k-block is 8 filter taps, K
        # padded to whole k-blocks (Wt [cout, ceil(k*k*8 / 64) * 64], zeros past k*k*8)
        kind, kd = "conv_fprop_c8_bf16_n64", (k * k * 8 + 63) // 64 * 64
    else:
        kind = "conv_fprop_bf16" + ("f32" if out.dtype == torch.float32 else "") + ("" if cout % 128 == 0 else "_n64")
        kd = k * k * c
    g = _conv_geom(n, h, w, c, k, stride, pad)
    extra = () if bn is None else (None, None, None, C.addressof(bn.c))
    return DeviceKernel(kind, (x.data_ptr(), Wt.data_ptr(), out.data_ptr(), C.addressof(g)) + extra,
                        (P, cout, kd, 0, splits), keep=(x, Wt, out, g) + (() if bn is None else (bn,)))


def conv_wgrad(dy, x, gpart, n, h, w, c, k, stride, pad, splits: int = 1) -> DeviceKernel:
    """Implicit-GEMM weight gradient: dW[cout, k*k*c] (fp32 split-K partials
    [splits, cout, k*k*c]) = dy^T . im2col(x), dy [P, cout] read MN-major as
    stored, im2col(x) gathered by TMA im2col loads."""
    cout = dy.shape[1]
    ho = (h + 2 * pad - k) // stride + 1
    wo = (w + 2 * pad - k) // stride + 1
    P = n * ho * wo
    kd = k * k * c
    kind = "conv_wgrad_bf16f32" + ("" if kd % 128 == 0 and c % 128 == 0 else "_n64")
    if c == 8:   # 8-channel input: N = the k*k*8 taps padded to 64-wide tiles
        kind, kd = "conv_wgrad_c8_bf16f32_n64", (k * k * 8 + 63) // 64 * 64
    g = _conv_geom(n, h, w, c, k, stride, pad)
    return DeviceKernel(kind, (dy.data_ptr(), x.data_ptr(), gpart.data_ptr(), C.addressof(g)),
                        (cout, kd, P, 0, splits), keep=(dy, x, gpart, g))


def im2col(x, col, n, h, w, c, kh, kw, stride, pad) -> DeviceKernel:
    return DeviceKernel("im2col_bf16", (x, col), (n, h, w, c, _pack_conv(kh, kw, stride, pad)))


def col2im(col, dx, n, h, w, c, kh, kw, stride, pad) -> DeviceKernel:
    return DeviceKernel("col2im_bf16", (col, dx), (n, h, w, c, _pack_conv(kh, kw, stride, pad)))


def transpose(src, dst) -> DeviceKernel:
    R, Cc = src.shape
    return DeviceKernel("transpose_bf16", (src, dst), (R, Cc))


def bn_stats(x, part, P, C, rb, mean, invstd, gamma, beta=None, scale_shift=None, eps=1e-5) -> DeviceKernel:
    """Forward BN statistics, finalised in the same kernel: mean, invstd and
    scale_shift [2, C] (y = x*scale + shift)."""
    return DeviceKernel("bn_stats", (x, None, None, None, mean, invstd, part, gamma),
                        (P, C, 0, rb, _ptr(beta), _ptr(scale_shift)), (eps,), keep=(beta, scale_shift))


def bn_stats_bwd(x, g, part, P, C, rb, mean, invstd, gamma, dgamma, dbeta, coef, g2=None, y=None) -> DeviceKernel:
    """Backward BN statistics, finalised in the same kernel: dgamma, dbeta and
    coef [3, C] with dx = coef[0]*dz + coef[1]*x + coef[2], dz = (g [+ g2]) * (y > 0)."""
    return DeviceKernel("bn_stats_bwd", (x, g, g2, y, mean, invstd, part, gamma),
                        (P, C, 1, rb, _ptr(dgamma), _ptr(dbeta), _ptr(coef)), keep=(dgamma, dbeta, coef))


def splitk_reduce(parts, out, bias=None, res=None, pre=None, act=0) -> DeviceKernel:
    """out (bf16) = parts.sum(0) for fp32 split-K partials [S, ...].  With
    ``bias`` (fp32 [C], out a row-major [rows, C]): the fused linear-layer
    epilogue out = act(sum + bias (+ res)), ``pre`` receiving the
    pre-activation values (as ``bias_act``)."""
    C = out.shape[-1]
    ep = bias is not None or res is not None or pre is not None or act
    return DeviceKernel("splitk_reduce", (parts, out, bias, res, pre),
                        (out.numel(), parts.shape[0], C if ep else 0, act))


def splitk_reduce_bn(parts, out, bn: BnStatsOut) -> DeviceKernel:
    """out [P, C] (bf16) = parts.sum(0) (fp32 split-K partials [S, P, C]) and
    the training batch-norm statistics of out (bn_stats mode 0) in one pass;
    ``bn.c.rb`` rows per logical block."""
    S, P, Cc = parts.shape
    return DeviceKernel("splitk_reduce_bn", (parts, out, None, None, None, None, None, C.addressof(bn.c)),
                        (P, Cc, S), keep=(bn,))


def bn_fold(rows, R, Cn, count, bn: BnStatsOut) -> DeviceKernel:
    """Training batch-norm statistics from the partial rows [2, R, Cn] a GEMM /
    conv_fprop epilogue wrote through ``BnStatsOut`` (``rows`` = its part):
    mean, invstd and scale_shift of ``count`` output rows into ``bn`` (whose
    own part is this fold's scratch, ``bn.c.rb`` rows per logical block)."""
    return DeviceKernel("bn_fold", (rows, None, None, None, None, None, None, C.addressof(bn.c)),
                        (R, Cn, count), keep=(bn, rows))


def bn_finalize_fwd(part, nrb, C, count, gamma, beta, mean, invstd, scale, shift,
                    eps=1e-5) -> DeviceKernel:
    return DeviceKernel("bn_finalize", (part, gamma, beta, mean, invstd, scale, shift),
                        (nrb, C, 0, count), (eps,))


def bn_finalize_bwd(part, nrb, C, count, gamma, mean, invstd, dgamma, dbeta, ca, cb, cc) -> DeviceKernel:
    """Backward statistics -> dgamma, dbeta and bn_bwd's per-channel
    coefficients (dx = ca*dz + cb*x + cc)."""
    return DeviceKernel("bn_finalize", (part, gamma, mean, invstd, dgamma, dbeta, ca, cb),
                        (nrb, C, 1, count, _ptr(cc)), keep=(cc,))


def bn_act(x, y, scale, shift, P, C, relu=True, res=None) -> DeviceKernel:
    return DeviceKernel("bn_act", (x, res, y, scale, shift), (P, C, int(relu)))


def bn_bwd(g, x, ca, cb, cc, dx, P, C, g2=None, y=None, dz_out=None) -> DeviceKernel:
    """dz = (g [+ g2]) * (y > 0);  dx = ca*dz + cb*x + cc;  optional dz output."""
    return DeviceKernel("bn_bwd", (g, g2, y, x, ca, cb, cc, dx), (P, C, _ptr(dz_out) or 0),
                        keep=tuple(t for t in (dz_out,) if t is not None))


def maxpool_fwd(x, y, arg, n, h, w, c) -> DeviceKernel:
    return DeviceKernel("maxpool_fwd", (x, y, arg), (n, h, w, c))


def maxpool_bwd(dy, arg, dx, n, h, w, c, dy2=None) -> DeviceKernel:
    return DeviceKernel("maxpool_bwd", (dy, dy2, arg, dx), (n, h, w, c))


def avgpool_fwd(x, y, n, hw, c) -> DeviceKernel:
    return DeviceKernel("avgpool_fwd", (x, y), (n, hw, c))


def avgpool_bwd(dy, dx, n, hw, c) -> DeviceKernel:
    return DeviceKernel("avgpool_bwd", (dy, dx), (n, hw, c))


def softmax_xent(logits, bias, labels, loss, dl, dl32, ncls) -> DeviceKernel:
    """Per-row softmax cross-entropy over the first ``ncls`` of ``Npad``
    columns (Npad % 8 == 0): ``loss`` [B], ``dl`` [B, Npad] bf16 = (softmax -
    onehot) / B, optional fp32 copy ``dl32``.  ``logits`` fp32 or bf16;
    ``bias`` [Npad] fp32 or None."""
    import torch
    B, Npad = logits.shape
    return DeviceKernel("softmax_xent", (logits, bias, labels, loss, dl, dl32),
                        (B, Npad, ncls, int(logits.dtype == torch.bfloat16)))


def sgd_update(segs, blockmap, blocks, nbytes, lr, momentum) -> DeviceKernel:
    """``segs``: device tensor of packed SgdSeg records; ``blockmap``: int32
    [blocks, 2] (segment, chunk) pairs -- see resnet.SgdTable."""
    return DeviceKernel("sgd_update", (segs, blockmap), (blocks, int(nbytes)), (lr, momentum))


# -- best-effort transformer-training kinds (config C3, kernels_tf.cu) ---------
def bias_act(x, y, bias, P, C, act=0, res=None, pre=None) -> DeviceKernel:
    """y = act(x + bias [+ res]); act 0 none, 1 ReLU, 2 GELU (tanh), 3 GELU (erf); ``pre``
    receives the pre-activation values (GELU backward input)."""
    return DeviceKernel("bn_act", (x, res, y, None, bias, pre), (P, C, act))


def colstats(g, part, P, C, rb, dbeta, dgamma=None, x=None, mean=None, rstd=None, g2=None) -> DeviceKernel:
    """Column sums over rows, finalised in-kernel: dbeta = sum_r g (+ g2);
    with ``x``: dgamma = sum_r g * (x - mean[r]) * rstd[r] (LayerNorm)."""
    return DeviceKernel("colstats", (x, g, g2, None, mean, rstd, part, None),
                        (P, C, 2, rb, _ptr(dgamma) or 0, _ptr(dbeta)),
                        keep=tuple(t for t in (dgamma, dbeta) if t is not None))


def layernorm_fwd(x, y, gamma, beta, mean, rstd, eps=1e-5) -> DeviceKernel:
    rows, C = x.shape
    return DeviceKernel("layernorm_fwd", (x, y, gamma, beta, mean, rstd), (rows, C), (eps,))


def layernorm_bwd(dy, x, gamma, mean, rstd, dx, g2=None) -> DeviceKernel:
    rows, C = x.shape
    return DeviceKernel("layernorm_bwd", (dy, g2, x, gamma, mean, rstd, dx), (rows, C))


def gelu_bwd(g, pre, dx, erf=False) -> DeviceKernel:
    """dx = g * GELU'(pre): tanh approximation (GPT-2) or exact erf (BERT)."""
    return DeviceKernel("gelu_bwd_erf" if erf else "gelu_bwd", (g, pre, dx), (g.numel(), int(erf)))


def softmax_causal(s, p, T, scale, causal=True) -> DeviceKernel:
    """P = softmax(scale * S) per row of T keys; ``causal``: keys j <= i only."""
    return DeviceKernel("softmax_causal", (s, p), (s.shape[0], T, int(causal)), (scale,))


def softmax_causal_bwd(p, dp, ds, T, scale, causal=True) -> DeviceKernel:
    return DeviceKernel("softmax_causal_bwd", (p, dp, ds), (p.shape[0], T, int(causal)), (scale,))


def embedding_fwd(tok, wte, wpe, x, T) -> DeviceKernel:
    rows, C = x.shape
    return DeviceKernel("embedding_fwd", (tok, wte, wpe, x), (rows, T, C))


def embedding_bwd(tok, dx, dwte) -> DeviceKernel:
    rows, C = dx.shape
    return DeviceKernel("embedding_bwd", (tok, dx, dwte), (rows, C))
