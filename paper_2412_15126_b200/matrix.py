"""Square matrices packed row-major into the slots, and their rotation primitives.

Mirror of reference ``pkg/src/slotrank/matrix.py``: cell (i, j) of an N x N
matrix sits in slot i*N + j (reference ``matrix.py:1-13``); replicate /
sum / transpose each cost log2(N) rotations and masks are one plaintext
multiply.  On the B200 engine every rotation is a Galois automorphism plus
one hybrid key switch, so these log-depth fold chains are the rotation-bound
part of the pipelines.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

__all__ = ["MatrixLayout", "mask", "sum_axis", "replicate", "transpose_vector"]


@dataclass(frozen=True)
class MatrixLayout:
    """Power-of-two side ``n_dim`` hosted in ``slot_count`` slots (``matrix.py:27-45``)."""

    n_dim: int
    slot_count: int

    def __post_init__(self):
        side = self.n_dim
        if side < 1 or side & (side - 1):
            raise ValueError(f"matrix side must be a power of two, got {side}")
        if side * side > self.slot_count:
            raise ValueError(
                f"matrix of side {side} needs {side * side} slots, only {self.slot_count} available"
            )

    @property
    def steps(self) -> int:
        return self.n_dim.bit_length() - 1


def _axis_ok(axis: str):
    if axis not in ("row", "col"):
        raise ValueError(f"axis must be 'row' or 'col', got {axis!r}")


@lru_cache(maxsize=None)
def _line_mask(n_dim: int, slot_count: int, axis: str, k: int) -> np.ndarray:
    """0/1 plaintext selecting row k (axis="row") or column k."""
    grid = np.zeros((n_dim, n_dim))
    if axis == "row":
        grid[k, :] = 1.0
    else:
        grid[:, k] = 1.0
    out = np.zeros(slot_count)
    out[: n_dim * n_dim] = grid.ravel()
    out.setflags(write=False)
    return out


def mask(engine, x, layout: MatrixLayout, axis: str, k: int):
    """Zero every cell outside row/column ``k`` (one ct x pt multiply)."""
    _axis_ok(axis)
    if k < 0 or k >= layout.n_dim:
        raise IndexError(f"{axis} index {k} out of range for side {layout.n_dim}")
    return engine.mul_plain(
        x, _line_mask(layout.n_dim, layout.slot_count, axis, k), site=f"mask-{axis}-{k}"
    )


def _fold(engine, x, offsets):
    """acc <- acc + rotate(acc, o) for each offset, in order (the log-depth chain)."""
    acc = x
    for off in offsets:
        acc = engine.add(acc, engine.rotate(acc, off))
    return acc


def _unit(layout: MatrixLayout, axis: str) -> int:
    return layout.n_dim if axis == "row" else 1


def sum_axis(engine, x, layout: MatrixLayout, axis: str):
    """axis="row": column sums land in row 0; axis="col": row sums in column 0."""
    _axis_ok(axis)
    unit = _unit(layout, axis)
    acc = _fold(engine, x, [unit << i for i in range(layout.steps)])
    return mask(engine, acc, layout, axis, 0)


def replicate(engine, x, layout: MatrixLayout, axis: str):
    """Copy row 0 into every row (axis="row") or column 0 into every column.

    Everything outside the source row/column must already be zero.
    """
    _axis_ok(axis)
    unit = _unit(layout, axis)
    return _fold(engine, x, [-(unit << i) for i in range(layout.steps)])


def transpose_vector(engine, x, layout: MatrixLayout, direction: str):
    """Move a vector between row 0 and column 0 (``matrix.py:101-118``).

    Rotations by N(N-1)/2^i, i = 1..log2 N (right for row_to_col, left for
    col_to_row), then one mask -- the [28, 14, 7] trace at N = 8.
    """
    if direction == "row_to_col":
        sign, keep = -1, "col"
    elif direction == "col_to_row":
        sign, keep = 1, "row"
    else:
        raise ValueError(f"unknown transpose direction {direction!r}")
    side = layout.n_dim
    span = side * (side - 1)
    acc = _fold(engine, x, [sign * (span >> i) for i in range(1, layout.steps + 1)])
    return mask(engine, acc, layout, keep, 0)
