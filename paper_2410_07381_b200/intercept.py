"""Generic best-effort routing: any PyTorch training step as a Tally program.

The reference schedules a best-effort job as a pipeline of ``KernelWork``s,
running untransformable kernels "exempt" -- whole, untransformed (ref
``scheduler.py:345-349``).  The hand-written programs in
``resnet.py`` / ``gpt2.py`` / ``bert.py`` are such pipelines written by hand;
this module derives one from an unmodified PyTorch step function:

1. ``capture(step_fn, *args)`` runs the step once eagerly under a
   ``TorchDispatchMode`` and records every ATen call (forward, autograd
   backward and optimizer) with the tensors it read and produced.  Those
   tensors stay alive: the program is static, like a CUDA graph.
2. Dense contractions become this package's transformable tcgen05 GEMM
   kernels (Original / Sliced / PTB): ``aten.mm`` and ``aten.addmm`` on
   bf16 with a supported operand layout (A K-major or MN-major, B K-major or
   MN-major, not A MN-major with B K-major) and N, K multiples of 64, and
   ``aten.bmm`` on contiguous batches.  ``addmm``'s bias is added by the next
   exempt segment.  Elementwise ``add`` / ``mul`` / ``relu`` / ``gelu`` /
   ``silu`` (and their in-place forms) on same-shape contiguous fp32 / bf16
   tensors become the transformable ``ewise`` kind.
3. Every maximal run of other ops (elementwise, normalisation, softmax,
   reductions, optimizer foreach ops, copies) is captured into one CUDA graph
   that re-executes them on the recorded tensors (results copied into the
   recorded outputs, view ops skipped -- the recorded views alias static
   storage) and becomes one exempt ``cuda_graph`` step.

The result is a ``Program`` whose ``works()`` are ``KernelWork``s for
``TaskScript``: the profile-guided tuner shapes the GEMMs like any other
kernel, and the scheduler preempts them by flag; the exempt graphs run whole.
Requirements are those of CUDA-graph capture: the step must be graph-safe
(no host synchronisation, no data-dependent shapes, no CPU-side state the
replay would have to advance).
"""

from __future__ import annotations

import threading

import torch
from torch.utils._python_dispatch import TorchDispatchMode
from torch.utils._pytree import tree_flatten, tree_map

from . import kernels
from .scheduler import KernelWork

aten = torch.ops.aten
_GEMM_OPS = {aten.mm.default, aten.addmm.default, aten.bmm.default}
# elementwise ops -> the transformable `ewise` kind: (op, binary, in-place)
_EWISE_OPS = {
    aten.add.Tensor: ("add", True, False), aten.add_.Tensor: ("add", True, True),
    aten.mul.Tensor: ("mul", True, False), aten.mul_.Tensor: ("mul", True, True),
    aten.relu.default: ("relu", False, False), aten.relu_.default: ("relu", False, True),
    aten.silu.default: ("silu", False, False), aten.silu_.default: ("silu", False, True),
    aten.gelu.default: ("gelu", False, False),
}


class _Record:
    __slots__ = ("func", "args", "kwargs", "out")

    def __init__(self, func, args, kwargs, out):
        self.func, self.args, self.kwargs, self.out = func, args, kwargs, out


class _Recorder(TorchDispatchMode):
    """Records every ATen call in execution order (the autograd engine's
    worker thread inherits the mode, so backward ops are seen too)."""

    def __init__(self):
        super().__init__()
        self.records = []
        self._lock = threading.Lock()

    def __torch_dispatch__(self, func, types, args=(), kwargs=None):
        kwargs = kwargs or {}
        out = func(*args, **kwargs)
        with self._lock:
            self.records.append(_Record(func, args, kwargs, out))
        return out


def _cuda_tensors(x):
    return [t for t in tree_flatten(x)[0] if isinstance(t, torch.Tensor) and t.is_cuda]


def _mn_major(t):
    """2-D t stored transposed (column-major): t.t() is a row-major view."""
    return t.dim() == 2 and t.stride(0) == 1 and t.stride(1) >= t.shape[0]


def _k_major(t):
    return t.dim() == 2 and t.stride(1) == 1 and t.stride(0) >= t.shape[1]


def _gemm_kernel(rec):
    """The transformable kernel for a recorded mm / addmm / bmm, or None."""
    f = rec.func
    a = tuple(t.detach() if isinstance(t, torch.Tensor) else t for t in rec.args)
    if f is aten.bmm.default:
        X, Y = a
        out = rec.out.detach()
        if not (X.dtype == Y.dtype == out.dtype == torch.bfloat16 and X.is_contiguous() and Y.is_contiguous()
                and out.is_contiguous()):
            return None
        Bn, M, K = X.shape
        N = Y.shape[2]
        if K % 64 or N % 64 or M % 8:
            return None
        # C_z[M,N] = X_z[M,K] . Y_z[K,N]: A K-major, B MN-major (stored [K,N]); batch z moves rows
        return kernels.gemm_ex(X.view(Bn * M, K), Y.view(Bn * K, N), out.view(Bn * M, N), M, N, K,
                               a_mn=False, b_mn=True, batches=Bn,
                               a_off=((M, 0), (0, 0)), b_off=((K, 0), (0, 0)), c_off=((M, 0), (0, 0)))
    X, Y = (a[1], a[2]) if f is aten.addmm.default else (a[0], a[1])
    out = rec.out.detach()
    if f is aten.addmm.default and (rec.kwargs.get("beta", 1) != 1 or rec.kwargs.get("alpha", 1) != 1):
        return None
    if not (X.dtype == Y.dtype == out.dtype == torch.bfloat16 and out.is_contiguous() and out.dim() == 2):
        return None
    M, K = X.shape
    N = Y.shape[1]
    if K % 64 or N % 64 or M % 8:
        return None
    if _k_major(X):
        A, a_mn = X, False
    elif _mn_major(X):
        A, a_mn = X.t(), True
    else:
        return None
    if _mn_major(Y):
        B, b_mn = Y.t(), False          # Y = W^T of a row-major W[N,K] (nn.Linear)
    elif _k_major(Y):
        B, b_mn = Y, True               # Y row-major [K,N]
    else:
        return None
    if a_mn and not b_mn:
        return None                     # no A MN-major x B K-major kind
    return kernels.gemm_ex(A, B, out, M, N, K, a_mn=a_mn, b_mn=b_mn)


def _ewise_kernel(rec):
    """The transformable kernel for a recorded elementwise op on same-shape
    contiguous fp32 / bf16 tensors (no broadcasting, no type promotion), or None."""
    op, binary, inplace = _EWISE_OPS[rec.func]
    args = [t.detach() if isinstance(t, torch.Tensor) else t for t in rec.args]
    x = args[0]
    out = rec.out.detach() if isinstance(rec.out, torch.Tensor) else None
    if out is None or not isinstance(x, torch.Tensor) or x.dtype not in (torch.float32, torch.bfloat16):
        return None
    y = args[1] if binary and len(args) > 1 else None
    if binary and not (isinstance(y, torch.Tensor) and y.shape == x.shape and y.dtype == x.dtype
                       and y.is_contiguous()):
        return None
    alpha = float(rec.kwargs.get("alpha", 1.0))
    if op == "gelu":
        approx = rec.kwargs.get("approximate", args[1] if len(args) > 1 else "none")
        op = "gelu_tanh" if approx == "tanh" else "gelu"
    per = 8 if x.dtype == torch.bfloat16 else 4
    tensors = [x, out] + ([y] if y is not None else [])
    if (out.shape != x.shape or out.dtype != x.dtype or not x.is_contiguous() or not out.is_contiguous()
            or x.numel() % per or any(t.data_ptr() % 16 for t in tensors)):
        return None
    if inplace and out.data_ptr() != x.data_ptr():
        return None
    return kernels.ewise(op, x, y, out, alpha)


class Program:
    """A captured step: ``items`` in order, each ("gemm", DeviceKernel, record)
    or ("graph", DeviceKernel, records).  ``works(prefix)`` -> KernelWorks."""

    def __init__(self, items, records):
        self.items = items
        self.records = records          # keeps every recorded tensor alive

    def works(self, prefix="step"):
        out = []
        for i, (what, dk, _r) in enumerate(self.items):
            if what != "graph":
                kid = f"{prefix}.{i}:{dk.kind}:{dk.info.grid}"
                out.append(KernelWork(kid, dk.cost(), kernel=dk))
            else:
                out.append(KernelWork(f"{prefix}.{i}:graph", dk.cost(), exempt=True, kernel=dk))
        return tuple(out)

    @property
    def n_gemm(self):
        return sum(1 for w, _d, _r in self.items if w == "gemm")

    @property
    def n_ewise(self):
        return sum(1 for w, _d, _r in self.items if w == "ewise")

    def run_original(self, stream):
        """The program once, every step untransformed, in order."""
        for _w, dk, _r in self.items:
            dk.original(stream).wait()


def _replay(records):
    """Re-execute recorded non-view ops on the recorded tensors (inside a
    CUDA-graph capture), writing results into the recorded outputs."""
    for r in records:
        if r.func.is_view:
            continue
        # detached aliases: same storage, no autograd metadata (the replay is
        # data movement, not a differentiable program)
        det = lambda t: t.detach() if isinstance(t, torch.Tensor) else t   # noqa: E731
        res = r.func(*tree_map(det, r.args), **tree_map(det, r.kwargs))
        outs = tree_flatten(r.out)[0]
        got = tree_flatten(res)[0]
        for o, g in zip(outs, got):
            if isinstance(o, torch.Tensor) and isinstance(g, torch.Tensor) and o.is_cuda and \
                    o.data_ptr() != g.data_ptr():
                o.copy_(g)


def _bias_add(rec):
    """addmm's bias, added after the GEMM in the next exempt segment."""
    bias, out = rec.args[0], rec.out
    return _Record(aten.add_.Tensor, (out, bias), {}, out)


def capture(step_fn, *args, **kwargs) -> Program:
    """Run ``step_fn(*args, **kwargs)`` once (eagerly, with its real effects)
    and return the Tally program that re-executes it."""
    rec = _Recorder()
    with rec:
        step_fn(*args, **kwargs)
    torch.cuda.synchronize()
    with torch.no_grad():
        return _build(rec)


def _build(rec) -> Program:
    records = [r for r in rec.records if _cuda_tensors((r.args, r.kwargs, r.out))]
    items, segment = [], []
    side = torch.cuda.Stream()

    def flush():
        if not [r for r in segment if not r.func.is_view]:
            segment.clear()
            return
        g = torch.cuda.CUDAGraph()
        seg = list(segment)
        # capture only -- no warm-up replay: re-running the segment would
        # apply its in-place updates (optimizer) a second time
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(g, stream=side):
            _replay(seg)
        torch.cuda.synchronize()
        items.append(("graph", kernels.cuda_graph(g), seg))
        segment.clear()

    for r in records:
        dk = _gemm_kernel(r) if r.func in _GEMM_OPS else \
            _ewise_kernel(r) if r.func in _EWISE_OPS else None
        if dk is None:
            segment.append(r)
            continue
        flush()
        items.append(("gemm" if r.func in _GEMM_OPS else "ewise", dk, r))
        if r.func is aten.addmm.default:
            segment.append(_bias_add(r))
    flush()
    return Program(items, records)


__all__ = ["capture", "Program"]
