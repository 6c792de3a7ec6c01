"""Host side of the kernel transformation layer.

On the B200 the transformations are compiled into every kernel (the Sliced
and PTB instantiations in ``csrc/tally_device.cuh``); what remains on the host
is the tiling arithmetic the scheduler and the tuner share:

* :func:`slice_extents` -- ref ``transforms.py:136-152`` (``round`` is
  half-even; the last slice absorbs the remainder),
* :func:`slice_plan`    -- the sub-launch table of a sliced kernel: linear
  ``(offset, count)`` ranges over the x-fastest task order (the scheduler's
  1-D tiling, ref ``scheduler.py:377-390``) or, with ``grid=``, the
  reference's rectangular largest-axis plan (ref ``transforms.py:155-168``).
* :func:`has_unified_sync_shape` / :func:`unify_synchronization` -- the
  reference's unified-synchronisation pass (ref ``transforms.py:200-288``) for
  IR kernels the IR-JIT compiles (``irjit.py``); hand-written bodies have the
  shape by construction.
"""

from __future__ import annotations

from fractions import Fraction

from ._lib import TransformError

__all__ = ["TransformError", "slice_extents", "slice_plan", "linearize", "delinearize",
           "has_unified_sync_shape", "unify_synchronization"]


def slice_extents(axis_len: int, fraction) -> list:
    f = Fraction(fraction)
    if not 0 < f <= 1:
        raise TransformError(f"slice fraction must be in (0, 1], got {fraction}")
    ext = min(max(1, round(f * axis_len)), axis_len)
    out = [ext] * (axis_len // ext)
    out[-1] += axis_len % ext
    return out


def slice_plan(total_blocks: int, fraction, grid=None):
    """Linear plan: [(offset, count), ...].  With ``grid=(x, y, z)``: the
    rectangular plan [((ox, oy, oz), (sx, sy, sz)), ...] along the largest axis
    (ties x -> y -> z)."""
    if grid is None:
        out, off = [], 0
        for ext in slice_extents(total_blocks, fraction):
            out.append((off, ext))
            off += ext
        return out
    g = list(grid)
    axis = max(range(3), key=lambda a: (g[a], -a))
    out, off = [], 0
    for ext in slice_extents(g[axis], fraction):
        o, s = [0, 0, 0], list(g)
        o[axis], s[axis] = off, ext
        out.append((tuple(o), tuple(s)))
        off += ext
    return out


def linearize(idx, dims) -> int:
    """ref ir/core.py:52-56 (x fastest)."""
    x, y, z = idx
    X, Y, Z = dims
    if not (0 <= x < X and 0 <= y < Y and 0 <= z < Z):
        raise ValueError(f"index {idx} out of range for dims {dims}")
    return x + y * X + z * X * Y


def delinearize(task: int, dims) -> tuple:
    """ref ir/core.py:59-65."""
    X, Y, Z = dims
    if not 0 <= task < X * Y * Z:
        raise ValueError(f"task index {task} out of range for dims {dims}")
    return task % X, (task // X) % Y, task // (X * Y)


# ------------------------------------------------------- unified synchronisation
# Kernels here are in the IR-JIT's normalised form (``irjit.normalize``):
# {"name", "params", "nparams", "grid", "block", "regs", "shared", "dependent",
#  "body": [(opcode, operands, label)]}, operands ("r", i) / ("i", v) /
# ("s", kind, axis) / ("l", name).

def has_unified_sync_shape(k: dict) -> bool:
    """Exactly one RET, and it is the last instruction (ref transforms.py:200-207)."""
    body = k["body"]
    return sum(op == "RET" for op, _a, _l in body) == 1 and body[-1][0] == "RET"


def _fresh_names(k: dict):
    used = {lab for _o, _a, lab in k["body"] if lab is not None} | set(k.get("params", ()))
    counter = [0]

    def fresh(base: str) -> str:
        name = base
        while name in used:
            counter[0] += 1
            name = f"{base}_{counter[0]}"
        used.add(name)
        return name
    return fresh


def unify_synchronization(k: dict) -> dict:
    """Route every barrier and every return through one synchronisation hub
    (ref transforms.py:210-288), so that the PTB worker loop's barriers are the
    only ones a finished logical block can meet:

    * a ``BAR_SYNC`` becomes "remember resume site n; jump to the hub";
    * a ``RET`` becomes "mark returned; count it in a shared word; jump to the hub";
    * the hub: barrier; if every thread has returned, leave through the one
      terminal ``RET``; a returned thread waits at the hub again; the others
      resume at their recorded site.

    Two registers (returned flag, resume site) and two scratch registers are
    appended, and one shared word (the returned count).  The count is a
    load / add / store on one shared word -- the IR-JIT compiles that triple
    to one shared-memory atomic add, the only correct form when a warp's
    threads return together.  Output labels and register /
    shared numbering equal the reference pass's."""
    fresh = _fresh_names(k)
    hub, leave = fresh("__usync"), fresh("__uret")
    word = k["shared"]
    rc = k["regs"]
    r_ret, r_site, r_a, r_b = ("r", rc), ("r", rc + 1), ("r", rc + 2), ("r", rc + 3)
    bx, by, bz = k["block"]
    body = k["body"]

    resume = {}        # instruction index after a barrier -> its resume label
    sites = []
    for j, (op, _a, _lab) in enumerate(body):
        if op != "BAR_SYNC":
            continue
        nxt_lab = body[j + 1][2]
        if nxt_lab is not None:
            lab = nxt_lab
        elif j + 1 in resume:
            lab = resume[j + 1]
        else:
            lab = fresh(f"__u_res{len(sites) + 1}")
            resume[j + 1] = lab
        sites.append(lab)

    imm = lambda v: ("i", v)   # noqa: E731
    out = [("CONST", (r_ret, imm(0)), None), ("CONST", (r_site, imm(0)), None),
           ("STORE_SHARED", (imm(word), imm(0)), None), ("BAR_SYNC", (), None)]
    n = 0
    for j, (op, args, lab) in enumerate(body):
        lab = resume.get(j, lab)
        if op == "BAR_SYNC":
            n += 1
            out += [("CONST", (r_site, imm(n)), lab), ("JUMP", (("l", hub),), None)]
        elif op == "RET":
            out += [("CONST", (r_ret, imm(1)), lab), ("LOAD_SHARED", (r_a, imm(word)), None),
                    ("ADD", (r_a, r_a, imm(1)), None), ("STORE_SHARED", (imm(word), r_a), None),
                    ("JUMP", (("l", hub),), None)]
        else:
            out.append((op, args, lab))
    out += [("BAR_SYNC", (), hub), ("LOAD_SHARED", (r_a, imm(word)), None),
            ("CMP_EQ", (r_b, r_a, imm(bx * by * bz)), None), ("BRANCH", (r_b, ("l", leave)), None),
            ("BRANCH", (r_ret, ("l", hub)), None)]
    for no, lab in enumerate(sites, start=1):
        out += [("CMP_EQ", (r_b, r_site, imm(no)), None), ("BRANCH", (r_b, ("l", lab)), None)]
    out += [("JUMP", (("l", hub),), None), ("RET", (), leave)]
    u = dict(k)
    u.update(regs=rc + 4, shared=word + 1, body=out)
    return u
