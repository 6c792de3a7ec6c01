"""Oracle restatement of the reference IR->IR passes (``transforms.py``).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

* ``add_block_offset``      — ref ``transforms.py:92-133``
* ``slice_extents``         — ref ``transforms.py:136-152`` (half-even ``round``)
* ``slice_kernel``          — ref ``transforms.py:155-168`` (largest axis, ties x->y->z)
* ``run_sliced``            — ref ``transforms.py:171-197``
* ``has_unified_sync_shape``/``unify_synchronization`` — ref ``transforms.py:200-288``
* ``make_preemptible``      — ref ``transforms.py:291-401`` (leader flag-then-claim)
* ``ptb_launch_args``/``run_ptb`` — ref ``transforms.py:404-448``
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

from .kernel_ir import (AXES, COMPLETED, DEFAULT_STEP_LIMIT, Dim3, Imm, Kernel,
                        MemTrigger, Op, Reg, Result, Special, interpret)


class TransformError(ValueError):
    """ref ``transforms.py:27-28``."""


@dataclass(frozen=True)
class SlicedPlan:
    base: Kernel
    subs: tuple  # ((offset Dim3, sub_grid Dim3), ...)


@dataclass(frozen=True)
class PtbControl:
    counter_addr: int
    flag_addr: int
    total: int
    grid: Dim3


def _no_dependent(k: Kernel, what: str):
    if k.dependent:
        raise TransformError(f"{k.name}: {what} refused (inter-block dependent)")


class _Fresh:
    """Collision-free names over a kernel's labels and params."""

    def __init__(self, k: Kernel):
        self.taken = set(k.label_map()) | set(k.params)
        self.n = 0

    def __call__(self, base: str) -> str:
        cand = base
        while cand in self.taken:
            self.n += 1
            cand = f"{base}_{self.n}"
        self.taken.add(cand)
        return cand


def _copy_params_to(first_param: int, count: int, first_reg: int):
    return [Op("MOV", (Reg(first_reg + i), Reg(first_param + i)))
            for i in range(count)]


def add_block_offset(k: Kernel) -> Kernel:
    _no_dependent(k, "block offset")
    fresh = _Fresh(k)
    new_params = tuple(fresh(f"__off_{a}") for a in AXES)
    np_ = len(k.params)
    base = max(k.regs, np_ + 3)
    off = {a: base + i for i, a in enumerate(AXES)}
    body = _copy_params_to(np_, 3, base)
    for op in k.body:
        if op.opcode == "READ_SPECIAL" and op.args[1].kind == "blockIdx":
            dst = op.args[0]
            body.append(op)
            body.append(Op("ADD", (dst, dst, Reg(off[op.args[1].axis]))))
        elif op.opcode == "READ_SPECIAL" and op.args[1].kind == "gridDim":
            body.append(Op("CONST", (op.args[0], Imm(k.grid.axis(op.args[1].axis))),
                           op.label))
        else:
            body.append(op)
    return Kernel(k.name, k.params + new_params, k.grid, k.block, base + 3,
                  k.shared, tuple(body), False)


def slice_extents(axis_len: int, fraction) -> list:
    f = Fraction(fraction)
    if not (0 < f <= 1):
        raise TransformError(f"fraction {fraction} outside (0, 1]")
    ext = min(max(1, round(f * axis_len)), axis_len)
    out = [ext] * (axis_len // ext)
    out[-1] += axis_len % ext
    return out


def slice_kernel(k: Kernel, fraction) -> SlicedPlan:
    _no_dependent(k, "slicing")
    axis = "x"
    for a in ("y", "z"):
        if k.grid.axis(a) > k.grid.axis(axis):
            axis = a
    subs = []
    start = 0
    for ext in slice_extents(k.grid.axis(axis), fraction):
        o = {a: 0 for a in AXES}
        g = {a: k.grid.axis(a) for a in AXES}
        o[axis], g[axis] = start, ext
        subs.append((Dim3(**o), Dim3(**g)))
        start += ext
    return SlicedPlan(add_block_offset(k), tuple(subs))


def run_sliced(plan: SlicedPlan, args, memory, seed: int = 0,
               step_limit: int = DEFAULT_STEP_LIMIT) -> Result:
    mem = tuple(memory)
    total = 0
    for i, (o, g) in enumerate(plan.subs):
        r = interpret(plan.base.with_grid(g), tuple(args) + (o.x, o.y, o.z), mem,
                      seed + i, step_limit)
        total += r.steps
        if r.status != COMPLETED:
            return Result(r.status, None, total)
        mem = r.memory
    return Result(COMPLETED, mem, total)


def has_unified_sync_shape(k: Kernel) -> bool:
    return (sum(op.opcode == "RET" for op in k.body) == 1
            and k.body[-1].opcode == "RET")


def unify_synchronization(k: Kernel) -> Kernel:
    fresh = _Fresh(k)
    hub, leave = fresh("__usync"), fresh("__uret")
    ret_word = k.shared
    r_ret, r_site, r_a, r_b = k.regs, k.regs + 1, k.regs + 2, k.regs + 3
    nthreads = k.block.total

    # resume label of every instruction that follows a barrier
    resume_at: dict = {}
    site_labels = []
    for j, op in enumerate(k.body):
        if op.opcode != "BAR_SYNC":
            continue
        nxt = k.body[j + 1]
        if nxt.label is not None:
            lab = nxt.label
        elif j + 1 in resume_at:
            lab = resume_at[j + 1]
        else:
            lab = fresh(f"__u_res{len(site_labels) + 1}")
            resume_at[j + 1] = lab
        site_labels.append(lab)

    body = [Op("CONST", (Reg(r_ret), Imm(0))), Op("CONST", (Reg(r_site), Imm(0))),
            Op("STORE_SHARED", (Imm(ret_word), Imm(0))), Op("BAR_SYNC")]
    site = 0
    for j, op in enumerate(k.body):
        lab = resume_at.get(j, op.label)
        if op.opcode == "BAR_SYNC":
            site += 1
            body += [Op("CONST", (Reg(r_site), Imm(site)), lab), Op("JUMP", (hub,))]
        elif op.opcode == "RET":
            body += [Op("CONST", (Reg(r_ret), Imm(1)), lab),
                     Op("LOAD_SHARED", (Reg(r_a), Imm(ret_word))),
                     Op("ADD", (Reg(r_a), Reg(r_a), Imm(1))),
                     Op("STORE_SHARED", (Imm(ret_word), Reg(r_a))),
                     Op("JUMP", (hub,))]
        else:
            body.append(op.relabel(lab))
    body += [Op("BAR_SYNC", (), hub),
             Op("LOAD_SHARED", (Reg(r_a), Imm(ret_word))),
             Op("CMP_EQ", (Reg(r_b), Reg(r_a), Imm(nthreads))),
             Op("BRANCH", (Reg(r_b), leave)),
             Op("BRANCH", (Reg(r_ret), hub))]
    for no, lab in enumerate(site_labels, start=1):
        body += [Op("CMP_EQ", (Reg(r_b), Reg(r_site), Imm(no))),
                 Op("BRANCH", (Reg(r_b), lab))]
    body += [Op("JUMP", (hub,)), Op("RET", (), leave)]
    return Kernel(k.name, k.params, k.grid, k.block, k.regs + 4, k.shared + 1,
                  tuple(body), k.dependent)


def make_preemptible(k: Kernel, workers: Dim3, enforce_unified: bool = True) -> Kernel:
    """Returns the worker kernel (its ``grid`` is the worker grid)."""
    _no_dependent(k, "preemption")
    if min(workers.x, workers.y, workers.z) < 1:
        raise TransformError(f"empty worker grid {workers}")
    if enforce_unified and not has_unified_sync_shape(k):
        raise TransformError(f"{k.name}: needs unified synchronization first")
    fresh = _Fresh(k)
    loop, stop, fence, itr, out = (fresh(n) for n in
                                   ("__ploop", "__pstop", "__pfence", "__piter", "__pexit"))
    extra = tuple(fresh(n) for n in ("__ctr_addr", "__flag_addr", "__total"))
    np_ = len(k.params)
    rb = max(k.regs, np_ + 3)
    ctr, flag, tot, task, bx, by, bz, t1, lead = range(rb, rb + 9)
    bidx = {"x": bx, "y": by, "z": bz}
    slot = k.shared

    body = _copy_params_to(np_, 3, rb) + [
        Op("READ_SPECIAL", (Reg(t1), Special("threadIdx", "x")), loop),
        Op("READ_SPECIAL", (Reg(lead), Special("threadIdx", "y"))),
        Op("ADD", (Reg(t1), Reg(t1), Reg(lead))),
        Op("READ_SPECIAL", (Reg(lead), Special("threadIdx", "z"))),
        Op("ADD", (Reg(t1), Reg(t1), Reg(lead))),
        Op("CMP_NE", (Reg(lead), Reg(t1), Imm(0))),
        Op("BRANCH", (Reg(lead), fence)),
        Op("LOAD_GLOBAL", (Reg(t1), Reg(flag))),       # flag gates the claim
        Op("BRANCH", (Reg(t1), stop)),
        Op("ATOMIC_ADD_GLOBAL", (Reg(t1), Reg(ctr), Imm(1))),
        Op("STORE_SHARED", (Imm(slot), Reg(t1))),
        Op("JUMP", (fence,)),
        Op("CONST", (Reg(t1), Imm(-1)), stop),
        Op("STORE_SHARED", (Imm(slot), Reg(t1))),
        Op("BAR_SYNC", (), fence),
        Op("LOAD_SHARED", (Reg(task), Imm(slot))),
        Op("CMP_LT", (Reg(t1), Reg(task), Imm(0))),
        Op("BRANCH", (Reg(t1), out)),
        Op("CMP_LT", (Reg(t1), Reg(task), Reg(tot))),
        Op("CMP_EQ", (Reg(t1), Reg(t1), Imm(0))),
        Op("BRANCH", (Reg(t1), out)),
        Op("MOD", (Reg(bx), Reg(task), Imm(k.grid.x))),
        Op("DIV", (Reg(t1), Reg(task), Imm(k.grid.x))),
        Op("MOD", (Reg(by), Reg(t1), Imm(k.grid.y))),
        Op("DIV", (Reg(bz), Reg(t1), Imm(k.grid.y))),
    ]
    for op in k.body:
        if op.opcode == "READ_SPECIAL" and op.args[1].kind == "blockIdx":
            body.append(Op("MOV", (op.args[0], Reg(bidx[op.args[1].axis])), op.label))
        elif op.opcode == "READ_SPECIAL" and op.args[1].kind == "gridDim":
            body.append(Op("CONST", (op.args[0], Imm(k.grid.axis(op.args[1].axis))),
                           op.label))
        elif op.opcode == "RET":
            body.append(Op("JUMP", (itr,), op.label))
        else:
            body.append(op)
    body += [Op("BAR_SYNC", (), itr), Op("JUMP", (loop,)), Op("RET", (), out)]
    return Kernel(k.name, k.params + extra, workers, k.block, rb + 9, k.shared + 1,
                  tuple(body))


def ptb_launch_args(ctl: PtbControl, args, memory) -> tuple:
    for a in (ctl.counter_addr, ctl.flag_addr):
        if not 0 <= a < len(memory):
            raise TransformError(f"control word {a} outside memory")
    if ctl.counter_addr == ctl.flag_addr:
        raise TransformError("counter and flag must differ")
    return tuple(args) + (ctl.counter_addr, ctl.flag_addr, ctl.total)


def run_ptb(worker_kernel: Kernel, ctl: PtbControl, args, memory, seed: int = 0,
            step_limit: int = DEFAULT_STEP_LIMIT, preempt_at_count=None) -> Result:
    full_args = ptb_launch_args(ctl, args, memory)
    trig = ()
    if preempt_at_count is not None:
        trig = (MemTrigger(ctl.counter_addr, preempt_at_count, ctl.flag_addr, 1),)
    return interpret(worker_kernel, full_args, memory, seed, step_limit, trig)
