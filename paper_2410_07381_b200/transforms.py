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
"""

from __future__ import annotations

from fractions import Fraction

from ._lib import TransformError

__all__ = ["TransformError", "slice_extents", "slice_plan", "linearize", "delinearize"]


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
