"""Temporal meshes for the space-time discretisation.

Same operations and contract as the reference's `stfem.temporal_mesh`
(/root/reference/pkg/src/stfem/temporal_mesh.py: type :10-46, `uniform`
:49-56, `graded` :59-68, `refine_bisect` :71-77), plus what the FDM path needs
on top of it: the DoF times for P1 and for the P2-in-time extension
(one midpoint DoF per element, DoFs ordered by time, t_0 removed; SURVEY.md
App. B).
"""

from __future__ import annotations

import numpy as np


def _validated(bp) -> np.ndarray:
    arr = np.array(bp, dtype=np.float64, copy=True).ravel()
    if arr.size < 2 or arr[0] != 0.0:
        raise ValueError("temporal mesh must start at t = 0")
    if np.any(arr[1:] <= arr[:-1]):
        raise ValueError("breakpoints must be strictly increasing")
    arr.setflags(write=False)
    return arr


class TemporalMesh:
    """Breakpoints 0 = t_0 < ... < t_N = T (immutable)."""

    __slots__ = ("_bp",)

    def __init__(self, breakpoints):
        object.__setattr__(self, "_bp", _validated(breakpoints))

    def __setattr__(self, name, value):  # immutability, like a frozen record
        raise AttributeError("TemporalMesh is immutable")

    def __eq__(self, other):
        return isinstance(other, TemporalMesh) and np.array_equal(self._bp, other._bp)

    def __hash__(self):
        return hash(self._bp.tobytes())

    def __repr__(self):
        return f"TemporalMesh(N={self.num_elements}, T={self.terminal_time:g})"

    breakpoints = property(lambda self: self._bp)
    terminal_time = property(lambda self: float(self._bp[-1]))
    num_elements = property(lambda self: int(self._bp.size - 1))
    steps = property(lambda self: np.diff(self._bp))
    max_step = property(lambda self: float(np.diff(self._bp).max()))

    @property
    def num_dofs(self) -> int:
        """n_t for P1: one DoF per breakpoint except t_0."""
        return self.num_elements

    def dof_times(self, degree: int = 1) -> np.ndarray:
        """Times of the temporal DoFs (P1: t_1..t_N; P2: mid_1, t_1, mid_2, ...)."""
        bp = self._bp
        if degree == 1:
            return bp[1:].copy()
        if degree != 2:
            raise ValueError("temporal degree must be 1 or 2")
        out = np.empty(2 * self.num_elements)
        out[0::2] = 0.5 * (bp[:-1] + bp[1:])
        out[1::2] = bp[1:]
        return out


def _check(T, N):
    if not T > 0:
        raise ValueError("terminal time must be positive")
    if int(N) < 1:
        raise ValueError("need at least one element")


def uniform(terminal_time: float, num_elements: int) -> TemporalMesh:
    """t_l = T l / N (paper Eq. (8))."""
    _check(terminal_time, num_elements)
    return TemporalMesh(terminal_time * np.arange(num_elements + 1) / num_elements)


def graded(terminal_time: float, num_elements: int, exponent: float) -> TemporalMesh:
    """t_l = T (l/N)^q, q >= 1."""
    if exponent < 1:
        raise ValueError("grading exponent must be >= 1")
    _check(terminal_time, num_elements)
    frac = np.arange(num_elements + 1) / num_elements
    return TemporalMesh(terminal_time * frac ** exponent)


def refine_bisect(mesh: TemporalMesh) -> TemporalMesh:
    """Insert every interval midpoint, keeping the old breakpoints."""
    bp = mesh.breakpoints
    mids = 0.5 * (bp[:-1] + bp[1:])
    return TemporalMesh(np.insert(bp, np.arange(1, bp.size), mids))
