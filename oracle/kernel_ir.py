"""Oracle restatement of the reference kernel IR and its interpreter.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Restates:
* word arithmetic ``wrap_word``               — ref ``ir/core.py:17-20``
* ``Dim3`` / linearize / delinearize          — ref ``ir/core.py:27-65``
* operand kinds and the opcode signature table — ref ``ir/core.py:68-118``
* ``KernelDef`` validation rules               — ref ``ir/core.py:153-214``
* ``LaunchSpec`` / ``ExecResult``              — ref ``ir/core.py:217-251``
* the block-serialised, round-robin-thread interpreter with barrier
  divergence detection and ``MemTrigger``      — ref ``ir/interp.py:46-265``

Kernels are exchanged with the fixtures as JSON (``kernel_from_json`` /
``kernel_to_json``): ``{"name", "params", "grid", "block", "regs", "shared",
"dependent", "body": [[opcode, [operand...], label], ...]}`` where an operand
is ``{"r": i}``, ``{"i": v}``, ``{"s": "kind.axis"}`` or a bare label string.
"""

from __future__ import annotations

import random
from dataclasses import dataclass

MASK64 = (1 << 64) - 1


def wrap64(v: int) -> int:
    """Two's-complement wrap to int64 (ref ``ir/core.py:17-20``)."""
    v &= MASK64
    return v - (1 << 64) if v >> 63 else v


AXES = ("x", "y", "z")
SPECIAL_KINDS = ("blockIdx", "threadIdx", "gridDim", "blockDim")


@dataclass(frozen=True, order=True)
class Dim3:
    """Extent or index triple, x fastest (ref ``ir/core.py:27-49``)."""

    x: int
    y: int = 1
    z: int = 1

    def __post_init__(self):
        if min(self.x, self.y, self.z) < 0:
            raise ValueError(f"negative Dim3 component in {self}")

    @property
    def total(self) -> int:
        return self.x * self.y * self.z

    def axis(self, a: str) -> int:
        return {"x": self.x, "y": self.y, "z": self.z}[a]

    def __iter__(self):
        return iter((self.x, self.y, self.z))


def linearize(idx: Dim3, dims: Dim3) -> int:
    """3-D index -> task index ``x + y*X + z*X*Y`` (ref ``ir/core.py:52-56``)."""
    if idx.x >= dims.x or idx.y >= dims.y or idx.z >= dims.z:
        raise ValueError(f"{idx} outside {dims}")
    return (idx.z * dims.y + idx.y) * dims.x + idx.x


def delinearize(task: int, dims: Dim3) -> Dim3:
    """Inverse of :func:`linearize` (ref ``ir/core.py:59-65``)."""
    if task < 0 or task >= dims.total:
        raise ValueError(f"task {task} outside {dims}")
    q, x = divmod(task, dims.x)
    z, y = divmod(q, dims.y)
    return Dim3(x, y, z)


@dataclass(frozen=True)
class Reg:
    index: int


@dataclass(frozen=True)
class Imm:
    value: int


@dataclass(frozen=True)
class Special:
    kind: str
    axis: str

    def __post_init__(self):
        if self.kind not in SPECIAL_KINDS or self.axis not in AXES:
            raise ValueError(f"bad special register {self.kind}.{self.axis}")


# operand signature per opcode: d=dest register, v=value (reg|imm),
# s=special register, l=label  (ref ir/core.py:96-118)
SIGNATURES = {
    "CONST": "dv", "MOV": "dv",
    "ADD": "dvv", "SUB": "dvv", "MUL": "dvv", "DIV": "dvv", "MOD": "dvv",
    "CMP_LT": "dvv", "CMP_LE": "dvv", "CMP_EQ": "dvv", "CMP_NE": "dvv",
    "READ_SPECIAL": "ds",
    "LOAD_GLOBAL": "dv", "STORE_GLOBAL": "vv", "ATOMIC_ADD_GLOBAL": "dvv",
    "LOAD_SHARED": "dv", "STORE_SHARED": "vv",
    "BAR_SYNC": "", "BRANCH": "vl", "JUMP": "l", "RET": "",
}


@dataclass(frozen=True)
class Op:
    """One body line (ref ``ir/core.py:121-150``)."""

    opcode: str
    args: tuple = ()
    label: str | None = None

    def __post_init__(self):
        sig = SIGNATURES.get(self.opcode)
        if sig is None:
            raise ValueError(f"unknown opcode {self.opcode}")
        if len(sig) != len(self.args):
            raise ValueError(f"{self.opcode}: arity {len(self.args)} != {len(sig)}")
        want = {"d": (Reg,), "v": (Reg, Imm), "s": (Special,), "l": (str,)}
        for k, a in zip(sig, self.args):
            if not isinstance(a, want[k]):
                raise ValueError(f"{self.opcode}: operand {a!r} is not kind {k}")

    def relabel(self, label):
        return Op(self.opcode, self.args, label)


class KernelValidationError(ValueError):
    pass


@dataclass(frozen=True)
class Kernel:
    """IR kernel record + validation (ref ``ir/core.py:153-214``)."""

    name: str
    params: tuple
    grid: Dim3
    block: Dim3
    regs: int
    shared: int
    body: tuple
    dependent: bool = False

    def __post_init__(self):
        object.__setattr__(self, "params", tuple(self.params))
        object.__setattr__(self, "body", tuple(self.body))
        self._check()

    def _check(self):
        bad = KernelValidationError
        if not self.body:
            raise bad(f"{self.name}: empty body")
        for d in (self.grid, self.block):
            if min(d.x, d.y, d.z) < 1:
                raise bad(f"{self.name}: zero extent {d}")
        if self.regs < len(self.params):
            raise bad(f"{self.name}: fewer registers than params")
        if self.shared < 0:
            raise bad(f"{self.name}: negative shared size")
        if len(set(self.params)) != len(self.params):
            raise bad(f"{self.name}: duplicate params")
        seen = set()
        for op in self.body:
            if op.label is not None:
                if op.label in seen:
                    raise bad(f"{self.name}: duplicate label {op.label}")
                seen.add(op.label)
        for op in self.body:
            for k, a in zip(SIGNATURES[op.opcode], op.args):
                if k == "l" and a not in seen:
                    raise bad(f"{self.name}: undefined label {a}")
                if isinstance(a, Reg) and a.index >= self.regs:
                    raise bad(f"{self.name}: r{a.index} beyond {self.regs} registers")
        if self.body[-1].opcode not in ("RET", "JUMP"):
            raise bad(f"{self.name}: must end in RET or JUMP")

    def label_map(self) -> dict:
        return {op.label: i for i, op in enumerate(self.body) if op.label is not None}

    def with_grid(self, grid: Dim3) -> "Kernel":
        return Kernel(self.name, self.params, grid, self.block, self.regs,
                      self.shared, self.body, self.dependent)


COMPLETED = "Completed"
DIVERGENT_BARRIER = "DivergentBarrier"
STEP_LIMIT_EXCEEDED = "StepLimitExceeded"
MEMORY_FAULT = "MemoryFault"
DEFAULT_STEP_LIMIT = 10 ** 7


@dataclass(frozen=True)
class Result:
    """ref ``ir/core.py:240-251``."""

    status: str
    memory: tuple | None
    steps: int


@dataclass(frozen=True)
class MemTrigger:
    """One-shot async host store: when ``mem[watch]`` becomes ``value`` after a
    global write to ``watch``, set ``mem[store] = store_value``
    (ref ``ir/interp.py:46-51``, ``:112-124``)."""

    watch: int
    value: int
    store: int
    store_value: int


class _MemFault(Exception):
    pass


def _lower(kernel: Kernel):
    """Body -> list of (opcode, decoded operands)."""
    where = kernel.label_map()
    out = []
    for op in kernel.body:
        dec = []
        for a in op.args:
            if isinstance(a, Reg):
                dec.append(("r", a.index))
            elif isinstance(a, Imm):
                dec.append(("i", wrap64(a.value)))
            elif isinstance(a, Special):
                dec.append(("s", (a.kind, a.axis)))
            else:
                dec.append(("l", where[a]))
        out.append((op.opcode, dec))
    return out


def _cdiv(a, b):
    """C truncating division; x/0 == 0 (ref ``ir/interp.py:201-206``)."""
    if b == 0:
        return 0
    q = abs(a) // abs(b)
    return wrap64(q if (a < 0) == (b < 0) else -q)


def _cmod(a, b):
    """C remainder; x%0 == 0 (ref ``ir/interp.py:207-211``)."""
    if b == 0:
        return 0
    q = abs(a) // abs(b)
    q = q if (a < 0) == (b < 0) else -q
    return wrap64(a - b * q)


_ARITH = {
    "ADD": lambda a, b: wrap64(a + b),
    "SUB": lambda a, b: wrap64(a - b),
    "MUL": lambda a, b: wrap64(a * b),
    "DIV": _cdiv,
    "MOD": _cmod,
    "CMP_LT": lambda a, b: int(a < b),
    "CMP_LE": lambda a, b: int(a <= b),
    "CMP_EQ": lambda a, b: int(a == b),
    "CMP_NE": lambda a, b: int(a != b),
}

_RUN, _WAIT, _DONE = 0, 1, 2


def interpret(kernel: Kernel, args, memory, seed: int = 0,
              step_limit: int = DEFAULT_STEP_LIMIT, triggers=()) -> Result:
    """Execute every block; ref ``ir/interp.py:77-265``.

    Blocks run one at a time in ``random.Random(seed)``-shuffled order of the
    x-fastest block list; inside a block, runnable threads (x-fastest order)
    each run to their next BAR_SYNC/RET, round-robin, until the barrier
    releases (all waiting, none returned) or every thread returned.
    """
    if len(args) != len(kernel.params):
        raise ValueError(f"{kernel.name}: {len(args)} args for {len(kernel.params)} params")
    prog = _lower(kernel)
    mem = list(memory)
    size = len(mem)
    argv = [wrap64(a) for a in args]
    grid, blk = kernel.grid, kernel.block
    armed = list(triggers)
    steps = 0

    order = [Dim3(x, y, z) for z in range(grid.z) for y in range(grid.y)
             for x in range(grid.x)]
    random.Random(seed).shuffle(order)

    def after_global_write(addr):
        nonlocal armed
        keep = []
        for t in armed:
            if t.watch == addr and mem[addr] == t.value:
                if not 0 <= t.store < size:
                    raise _MemFault()
                mem[t.store] = wrap64(t.store_value)
            else:
                keep.append(t)
        armed = keep

    def gaddr(a):
        if a < 0 or a >= size:
            raise _MemFault()
        return a

    threads = [(tx, ty, tz) for tz in range(blk.z) for ty in range(blk.y)
               for tx in range(blk.x)]
    try:
        for b in order:
            special = {("gridDim", "x"): grid.x, ("gridDim", "y"): grid.y,
                       ("gridDim", "z"): grid.z, ("blockDim", "x"): blk.x,
                       ("blockDim", "y"): blk.y, ("blockDim", "z"): blk.z,
                       ("blockIdx", "x"): b.x, ("blockIdx", "y"): b.y,
                       ("blockIdx", "z"): b.z}
            smem = [0] * kernel.shared
            regs = []
            for _ in threads:
                r = [0] * kernel.regs
                r[:len(argv)] = argv
                regs.append(r)
            pc = [0] * len(threads)
            state = [_RUN] * len(threads)

            while True:
                progressed = False
                for t, (tx, ty, tz) in enumerate(threads):
                    if state[t] != _RUN:
                        continue
                    progressed = True
                    R = regs[t]
                    p = pc[t]
                    mine = {("threadIdx", "x"): tx, ("threadIdx", "y"): ty,
                            ("threadIdx", "z"): tz}

                    def val(o):
                        return R[o[1]] if o[0] == "r" else o[1]

                    while True:
                        opc, ops = prog[p]
                        steps += 1
                        if steps > step_limit:
                            return Result(STEP_LIMIT_EXCEEDED, None, steps)
                        p += 1
                        if opc == "BAR_SYNC":
                            state[t] = _WAIT
                            break
                        if opc == "RET":
                            state[t] = _DONE
                            break
                        if opc == "JUMP":
                            p = ops[0][1]
                        elif opc == "BRANCH":
                            if val(ops[0]) != 0:
                                p = ops[1][1]
                        elif opc == "READ_SPECIAL":
                            key = ops[1][1]
                            R[ops[0][1]] = mine[key] if key in mine else special[key]
                        elif opc in ("CONST", "MOV"):
                            R[ops[0][1]] = val(ops[1])
                        elif opc in _ARITH:
                            R[ops[0][1]] = _ARITH[opc](val(ops[1]), val(ops[2]))
                        elif opc == "LOAD_GLOBAL":
                            R[ops[0][1]] = mem[gaddr(val(ops[1]))]
                        elif opc == "STORE_GLOBAL":
                            a = gaddr(val(ops[0]))
                            mem[a] = val(ops[1])
                            after_global_write(a)
                        elif opc == "ATOMIC_ADD_GLOBAL":
                            a = gaddr(val(ops[1]))
                            old = mem[a]
                            mem[a] = wrap64(old + val(ops[2]))
                            R[ops[0][1]] = old
                            after_global_write(a)
                        elif opc == "LOAD_SHARED":
                            a = val(ops[1])
                            if a < 0 or a >= kernel.shared:
                                raise _MemFault()
                            R[ops[0][1]] = smem[a]
                        elif opc == "STORE_SHARED":
                            a = val(ops[0])
                            if a < 0 or a >= kernel.shared:
                                raise _MemFault()
                            smem[a] = val(ops[1])
                        else:  # pragma: no cover
                            raise AssertionError(opc)
                    pc[t] = p
                if all(s == _DONE for s in state):
                    break
                if not progressed:
                    if _DONE in state:
                        return Result(DIVERGENT_BARRIER, None, steps)
                    state = [_RUN] * len(threads)
    except _MemFault:
        return Result(MEMORY_FAULT, None, steps)
    return Result(COMPLETED, tuple(mem), steps)


# -- fixture (de)serialisation ----------------------------------------------

def _operand_from_json(o):
    if isinstance(o, str):
        return o
    if "r" in o:
        return Reg(o["r"])
    if "i" in o:
        return Imm(o["i"])
    kind, axis = o["s"].split(".")
    return Special(kind, axis)


def _operand_to_json(a):
    if isinstance(a, Reg):
        return {"r": a.index}
    if isinstance(a, Imm):
        return {"i": a.value}
    if isinstance(a, Special):
        return {"s": f"{a.kind}.{a.axis}"}
    return a


def kernel_from_json(d) -> Kernel:
    return Kernel(
        name=d["name"], params=tuple(d["params"]), grid=Dim3(*d["grid"]),
        block=Dim3(*d["block"]), regs=d["regs"], shared=d["shared"],
        body=tuple(Op(o[0], tuple(_operand_from_json(a) for a in o[1]), o[2])
                   for o in d["body"]),
        dependent=bool(d.get("dependent", False)))


def kernel_to_json(k: Kernel) -> dict:
    return {"name": k.name, "params": list(k.params), "grid": list(k.grid),
            "block": list(k.block), "regs": k.regs, "shared": k.shared,
            "dependent": k.dependent,
            "body": [[o.opcode, [_operand_to_json(a) for a in o.args], o.label]
                     for o in k.body]}
