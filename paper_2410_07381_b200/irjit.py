"""IR -> CUDA JIT: any reference IR kernel in the three Tally launch shapes.

The reference's kernel transformer rewrites device code (§4.1); its
`tallysim` restates that on a mini SIMT IR (ref ``ir/core.py``,
``transforms.py``).  This module compiles such an IR kernel -- a reference
``KernelDef``, the oracle's ``Kernel``, or the fixtures' JSON encoding -- into
a CUDA *body* and instantiates it with the same ``k_original`` / ``k_sliced``
/ ``k_ptb`` templates every hand-written kernel uses (``csrc/tally_device.cuh``),
through NVRTC, for sm_100a:

* registers  -> a per-thread ``long long r[regs]`` (params in the low ones);
* global memory -> the launch's flat int64 word image (bounds-checked;
  a fault sets the fault word, like the interpreter's MemoryFault);
* shared memory -> zero-initialised per logical block (interpreter semantics);
* ``blockIdx`` -> the *logical* block (offset / delinearised task);
  ``gridDim`` -> the logical grid (the pinned extents of ref transforms.py:115-121);
* ``BAR_SYNC`` -> ``__syncthreads``; ``RET`` -> leave the body (in PTB shape
  the worker loop's end-of-iteration barrier is next);
* arithmetic wraps at 64 bits; DIV/MOD truncate, x/0 = x%0 = 0
  (ref ir/interp.py:195-211);
* a backward-branch budget stands in for the interpreter's step limit, so a
  non-terminating kernel faults instead of hanging the GPU.

PTB shape requires the unified-synchronisation shape the reference enforces
(ref transforms.py:310-314): a ``RET`` may not be followed by a reachable
``BAR_SYNC``.  Kernels violating it raise ``TransformError`` -- run them
through ``unify_synchronization`` first, exactly as the reference does.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import os

from . import _lib
from .device import B200Device
from .kernels import DeviceKernel
from .transforms import TransformError

_HERE = os.path.dirname(os.path.abspath(__file__))
_HEADER = os.path.join(_HERE, "csrc", "tally_device.cuh")
STEP_BUDGET = 1 << 22          # backward branches per thread before a fault


# -------------------------------------------------------------- normalise
def _norm_operand(o):
    """-> ('r', i) | ('i', v) | ('s', kind, axis) | ('l', name)."""
    if isinstance(o, str):
        return ("l", o)
    if isinstance(o, dict):
        if "r" in o:
            return ("r", int(o["r"]))
        if "i" in o:
            return ("i", int(o["i"]))
        kind, axis = o["s"].split(".")
        return ("s", kind, axis)
    if hasattr(o, "index"):
        return ("r", int(o.index))
    if hasattr(o, "value"):
        return ("i", int(o.value))
    if hasattr(o, "kind") and hasattr(o, "axis"):
        return ("s", o.kind, o.axis)
    raise TypeError(f"unknown IR operand {o!r}")


def normalize(kernel) -> dict:
    """Accept a reference KernelDef, an oracle Kernel, the JSON encoding, or
    an already normalised kernel (e.g. ``transforms.unify_synchronization``'s
    output)."""
    if isinstance(kernel, dict) and "nparams" in kernel:
        return kernel
    if isinstance(kernel, dict):
        d = kernel
        body = [(op, tuple(_norm_operand(a) for a in args), lab) for op, args, lab in d["body"]]
        return {"name": d["name"], "params": tuple(d["params"]), "nparams": len(d["params"]),
                "grid": tuple(d["grid"]), "block": tuple(d["block"]), "regs": d["regs"],
                "shared": d["shared"], "dependent": bool(d.get("dependent", False)), "body": body}
    regs = getattr(kernel, "register_count", None)
    regs = kernel.regs if regs is None else regs
    shared = getattr(kernel, "shared_words", None)
    shared = kernel.shared if shared is None else shared
    ops = []
    for ins in kernel.body:
        args = getattr(ins, "operands", None)
        args = ins.args if args is None else args
        ops.append((ins.opcode, tuple(_norm_operand(a) for a in args), ins.label))
    dep = getattr(kernel, "inter_block_dependent", None)
    dep = getattr(kernel, "dependent", False) if dep is None else dep
    return {"name": kernel.name, "params": tuple(kernel.params), "nparams": len(kernel.params),
            "grid": tuple(kernel.grid),
            "block": tuple(kernel.block), "regs": regs, "shared": shared, "dependent": bool(dep),
            "body": ops}


def ptb_safe(k: dict) -> bool:
    """No BAR_SYNC after a non-terminal RET in program order (a conservative,
    structural version of ref transforms.py:200-207, 310-314)."""
    body = k["body"]
    seen_ret = False
    for i, (op, _a, _l) in enumerate(body):
        if op == "RET" and i != len(body) - 1:
            seen_ret = True
        elif op == "BAR_SYNC" and seen_ret:
            return False
    return True


# -------------------------------------------------------------- codegen
def _val(o):
    if o[0] == "r":
        return f"r[{o[1]}]"
    if o[0] == "i":
        return f"{o[1]}LL" if o[1] != -(1 << 63) else "(-9223372036854775807LL - 1)"
    raise ValueError(f"not a value operand: {o}")


def _special(kind, axis, k):
    bx, by, bz = k["block"]
    if kind == "blockIdx":
        return f"(long long)bidx.{axis}"
    if kind == "gridDim":
        return f"(long long)grid.{axis}"
    if kind == "blockDim":
        return str({"x": bx, "y": by, "z": bz}[axis])
    return {"x": "tx", "y": "ty", "z": "tz"}[axis]


def _shared_increment(body, i, targets) -> bool:
    """body[i:i+3] == LOAD_SHARED rX, [W]; ADD rX, rX, 1; STORE_SHARED [W], rX
    with W an immediate and no branch target inside."""
    if i + 2 >= len(body) or (i + 1) in targets or (i + 2) in targets:
        return False
    (o0, a0, _), (o1, a1, _), (o2, a2, _) = body[i], body[i + 1], body[i + 2]
    if o1 != "ADD" or o2 != "STORE_SHARED" or a0[1][0] != "i":
        return False
    rx, w = a0[0], a0[1]
    return (a1[0] == rx and a1[1] == rx and a1[2] == ("i", 1) and a2[0] == w and a2[1] == rx)


def codegen(k: dict, ns: str) -> str:
    bx, by, bz = k["block"]
    threads = bx * by * bz
    labels = {lab: i for i, (_o, _a, lab) in enumerate(k["body"]) if lab is not None}
    L = []
    emit = L.append
    emit(f"namespace {ns} {{")
    emit("struct Body {")
    emit(f"  static constexpr int kThreads = {threads};")
    emit("  typedef tally::JitParams Params;")
    emit("  static __device__ __forceinline__ long long wdiv(long long a, long long b) {")
    emit("    if (b == 0) return 0; if (b == -1) return (long long)(0ull - (unsigned long long)a); return a / b; }")
    emit("  static __device__ __forceinline__ long long wmod(long long a, long long b) {")
    emit("    if (b == 0 || b == -1) return 0; return a % b; }")
    emit("  static __device__ void run(const Params& p, uint3 bidx, uint3 grid, char* smem_raw) {")
    emit("    long long* sh = reinterpret_cast<long long*>(smem_raw);")
    if k["shared"]:
        emit(f"    for (int i = threadIdx.x; i < {k['shared']}; i += kThreads) sh[i] = 0;")
        emit("    __syncthreads();")
    emit("    const int tid = threadIdx.x;")
    emit(f"    const long long tx = tid % {bx}, ty = (tid / {bx}) % {by}, tz = tid / {bx * by};")
    emit(f"    long long r[{max(1, k['regs'])}];")
    emit(f"    #pragma unroll\n    for (int i = 0; i < {max(1, k['regs'])}; ++i) r[i] = 0;")
    for i in range(k["nparams"]):
        emit(f"    r[{i}] = p.args[{i}];")
    emit("    unsigned long long budget = 0;")
    emit("    (void)sh; (void)tx; (void)ty; (void)tz; (void)budget; (void)bidx; (void)grid;")

    def goto(target, here):
        t = labels[target]
        if t <= here:   # backward branch: spend budget
            return (f"{{ if (++budget > {STEP_BUDGET}ull) {{ atomicOr(p.fault, 2ull); goto L_ret; }} "
                    f"goto L{t}; }}")
        return f"goto L{t};"

    targets = {labels[a[-1][1]] for op, a, _l in k["body"] if op in ("BRANCH", "JUMP")}
    body = k["body"]
    fused = set()
    for i, (op, a, _lab) in enumerate(body):
        if i in targets:
            emit(f"  L{i}:")
        if i in fused:
            continue
        if op == "LOAD_SHARED" and _shared_increment(body, i, targets):
            # load / add 1 / store back on one shared word (the unified-sync
            # returned count): one atomic, or a warp returning together would
            # count once
            w = a[1][1]
            emit(f"    {{ if ({w} < 0 || {w} >= {k['shared']}) {{ atomicOr(p.fault, 1ull); }} else "
                 f"r[{a[0][1]}] = (long long)atomicAdd(reinterpret_cast<unsigned long long*>(sh + {w}), 1ull) + 1; }}")
            fused.update((i + 1, i + 2))
            continue
        if op in ("CONST", "MOV"):
            emit(f"    r[{a[0][1]}] = {_val(a[1])};")
        elif op in ("ADD", "SUB", "MUL"):
            c = {"ADD": "+", "SUB": "-", "MUL": "*"}[op]
            emit(f"    r[{a[0][1]}] = (long long)((unsigned long long){_val(a[1])} {c} "
                 f"(unsigned long long){_val(a[2])});")
        elif op == "DIV":
            emit(f"    r[{a[0][1]}] = wdiv({_val(a[1])}, {_val(a[2])});")
        elif op == "MOD":
            emit(f"    r[{a[0][1]}] = wmod({_val(a[1])}, {_val(a[2])});")
        elif op.startswith("CMP_"):
            c = {"CMP_LT": "<", "CMP_LE": "<=", "CMP_EQ": "==", "CMP_NE": "!="}[op]
            emit(f"    r[{a[0][1]}] = ({_val(a[1])} {c} {_val(a[2])}) ? 1 : 0;")
        elif op == "READ_SPECIAL":
            emit(f"    r[{a[0][1]}] = {_special(a[1][1], a[1][2], k)};")
        elif op == "LOAD_GLOBAL":
            emit(f"    {{ const long long ad = {_val(a[1])}; if (ad < 0 || ad >= p.nwords) "
                 f"{{ atomicOr(p.fault, 1ull); }} else r[{a[0][1]}] = p.mem[ad]; }}")
        elif op == "STORE_GLOBAL":
            emit(f"    {{ const long long ad = {_val(a[0])}; if (ad < 0 || ad >= p.nwords) "
                 f"{{ atomicOr(p.fault, 1ull); }} else p.mem[ad] = {_val(a[1])}; }}")
        elif op == "ATOMIC_ADD_GLOBAL":
            emit(f"    {{ const long long ad = {_val(a[1])}; if (ad < 0 || ad >= p.nwords) "
                 f"{{ atomicOr(p.fault, 1ull); }} else r[{a[0][1]}] = (long long)atomicAdd("
                 f"reinterpret_cast<unsigned long long*>(p.mem + ad), "
                 f"(unsigned long long){_val(a[2])}); }}")
        elif op == "LOAD_SHARED":
            emit(f"    {{ const long long ad = {_val(a[1])}; if (ad < 0 || ad >= {k['shared']}) "
                 f"{{ atomicOr(p.fault, 1ull); }} else r[{a[0][1]}] = sh[ad]; }}")
        elif op == "STORE_SHARED":
            emit(f"    {{ const long long ad = {_val(a[0])}; if (ad < 0 || ad >= {k['shared']}) "
                 f"{{ atomicOr(p.fault, 1ull); }} else sh[ad] = {_val(a[1])}; }}")
        elif op == "BAR_SYNC":
            emit("    __syncthreads();")
        elif op == "BRANCH":
            emit(f"    if ({_val(a[0])} != 0) {goto(a[1][1], i)}")
        elif op == "JUMP":
            emit(f"    {goto(a[0][1], i)}")
        elif op == "RET":
            emit("    goto L_ret;")
        else:
            raise ValueError(f"unknown opcode {op}")
    emit("  L_ret:")
    emit("    return;")
    emit("  }")
    emit("};")
    emit("}")
    return "\n".join(L) + "\n"


# -------------------------------------------------------------- NVRTC
class _Nvrtc:
    def __init__(self):
        for name in ("libnvrtc.so.12", "libnvrtc.so"):
            try:
                self.lib = C.CDLL(name)
                break
            except OSError:
                continue
        else:
            raise ImportError("libnvrtc not found")
        L = self.lib
        L.nvrtcCreateProgram.argtypes = [C.POINTER(C.c_void_p), C.c_char_p, C.c_char_p, C.c_int,
                                         C.POINTER(C.c_char_p), C.POINTER(C.c_char_p)]
        L.nvrtcAddNameExpression.argtypes = [C.c_void_p, C.c_char_p]
        L.nvrtcCompileProgram.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_char_p)]
        L.nvrtcGetProgramLogSize.argtypes = [C.c_void_p, C.POINTER(C.c_size_t)]
        L.nvrtcGetProgramLog.argtypes = [C.c_void_p, C.c_char_p]
        L.nvrtcGetLoweredName.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_char_p)]
        L.nvrtcGetCUBINSize.argtypes = [C.c_void_p, C.POINTER(C.c_size_t)]
        L.nvrtcGetCUBIN.argtypes = [C.c_void_p, C.c_char_p]
        L.nvrtcDestroyProgram.argtypes = [C.POINTER(C.c_void_p)]

    def compile(self, src: str, name: str, exprs):
        L = self.lib
        hdr_src = open(_HEADER).read().encode()
        prog = C.c_void_p()
        hs = (C.c_char_p * 1)(hdr_src)
        hn = (C.c_char_p * 1)(b"tally_device.cuh")
        if L.nvrtcCreateProgram(C.byref(prog), src.encode(), name.encode(), 1, hs, hn) != 0:
            raise RuntimeError("nvrtcCreateProgram failed")
        try:
            for e in exprs:
                L.nvrtcAddNameExpression(prog, e.encode())
            opts = [b"-arch=sm_100a", b"-std=c++17", b"-default-device"]
            rc = L.nvrtcCompileProgram(prog, len(opts), (C.c_char_p * len(opts))(*opts))
            n = C.c_size_t()
            L.nvrtcGetProgramLogSize(prog, C.byref(n))
            log = C.create_string_buffer(n.value)
            L.nvrtcGetProgramLog(prog, log)
            if rc != 0:
                raise TransformError(f"NVRTC failed for {name}:\n{log.value.decode()}")
            lowered = []
            for e in exprs:
                out = C.c_char_p()
                L.nvrtcGetLoweredName(prog, e.encode(), C.byref(out))
                lowered.append(out.value.decode())
            L.nvrtcGetCUBINSize(prog, C.byref(n))
            cubin = C.create_string_buffer(n.value)
            L.nvrtcGetCUBIN(prog, cubin)
            return cubin, lowered
        finally:
            L.nvrtcDestroyProgram(C.byref(prog))


_nvrtc = None
_kinds: dict = {}
_images: list = []   # registered cubins stay alive: the runtime caches one module per image address


def _prepare(kernel):
    k = normalize(kernel)
    if k["dependent"]:
        raise TransformError(f"{k['name']}: inter-block dependent kernels are exempt")
    if k["nparams"] > 7:
        raise TransformError(f"{k['name']}: at most 7 IR parameters")
    digest = hashlib.sha256(repr(sorted((kk, str(v)) for kk, v in k.items())).encode()).hexdigest()[:16]
    return k, digest


def _compile_register(items):
    """items: [(normalised kernel, digest)] -> kind ids, one NVRTC program and
    one module for all of them."""
    global _nvrtc
    B200Device.get()
    if _nvrtc is None:
        _nvrtc = _Nvrtc()
    src = ['#include "tally_device.cuh"\n']
    exprs = []
    for k, digest in items:
        ns = f"tally_jit_{digest}"
        src.append(codegen(k, ns))
        exprs += [f"tally::k_original<{ns}::Body>", f"tally::k_sliced<{ns}::Body>", f"tally::k_ptb<{ns}::Body>"]
    cubin, lowered = _nvrtc.compile("".join(src), f"tally_jit_{items[0][1]}_x{len(items)}.cu", exprs)
    _images.append(cubin)
    ids = []
    for i, (k, digest) in enumerate(items):
        gx, gy, gz = k["grid"]
        bx, by, bz = k["block"]
        out = C.c_int()
        _lib.check(_lib.lib.tally_jit_register(f"ir_{digest}".encode(), C.cast(cubin, C.c_void_p),
                                               *[x.encode() for x in lowered[3 * i:3 * i + 3]], gx, gy, gz,
                                               bx * by * bz, 8 * k["shared"], C.byref(out)),
                   "jit register")
        _kinds[f"ir_{digest}"] = out.value
        ids.append(out.value)
    return ids


class JitKernel:
    """A compiled IR kernel kind; ``bind`` it to a memory image to launch."""

    def __init__(self, kernel, _prepared=None):
        k, digest = _prepared or _prepare(kernel)
        self.ir = k
        self.ptb_ok = ptb_safe(k)
        self.kind_name = f"ir_{digest}"
        if self.kind_name not in _kinds:
            _compile_register([(k, digest)])
        self.kind_id = _kinds[self.kind_name]

    @classmethod
    def compile_many(cls, kernels, chunk: int = 64) -> list:
        """Compile many IR kernels with one NVRTC program per ``chunk`` of them
        (the acceptance gate's 400 kinds in a few programs instead of 400)."""
        prepared = [_prepare(k) for k in kernels]
        todo, seen = [], set()
        for k, d in prepared:
            if f"ir_{d}" not in _kinds and d not in seen:
                seen.add(d)
                todo.append((k, d))
        for i in range(0, len(todo), chunk):
            _compile_register(todo[i:i + chunk])
        return [cls(None, p) for p in prepared]

    def bind(self, mem, fault, args) -> DeviceKernel:
        """mem: int64 CUDA tensor (the word image); fault: int64 CUDA tensor [1]."""
        dk = DeviceKernel(self.kind_name, (mem, fault), (mem.numel(),) + tuple(args))
        if not self.ptb_ok:
            orig_ptb = dk.ptb

            def refuse(*a, **kw):
                raise TransformError(f"{self.ir['name']}: preemption requires unified "
                                     "synchronization (RET before a barrier)")
            dk.ptb = refuse
            dk._unsafe_ptb = orig_ptb
        return dk
