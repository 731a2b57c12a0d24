"""Temporal core and its eigendecomposition — host fp64 one-off setup.

SPEC.md:230-310 (`dense_complex_linalg`).  The n_t x n_t problem is tiny next
to the space-time solve (n_t <= 1024) and the north star fixes it on the host
in fp64 "exactly as the reference does": LAPACK zgeev through scipy, unit
2-norm eigenvector columns, first nonzero component rotated to the positive
real axis, eigenvalues ordered by real then imaginary part
(:301), near-defect check sigma_min(X) < 1e-12 (:300), Y = X^{-1} (i B_t)^{-1}
by dense LU (:266, :281-289), kappa_2 = sigma_max / sigma_min (:272-280).
Timed separately from the solve as `t_setup`.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.linalg as sla


class NotDiagonalizable(np.linalg.LinAlgError):
    """caller should fall back to Bartels-Stewart."""


class DecompositionFailure(np.linalg.LinAlgError):
    """SPEC.md:252 singular B_t / :268 non-convergence."""


@dataclass(frozen=True)
class TemporalFactors:
    """X (transformation), S (diagonal eigenvalues for the
    eigen variant), Y = X^{-1}(iB_t)^{-1}, kappa2 = cond_2(X)."""

    X: np.ndarray
    S: np.ndarray
    Y: np.ndarray
    kappa2: float
    variant: str = "eigen"

    @property
    def eigenvalues(self) -> np.ndarray:
        return np.diag(self.S).copy()


def dense_solve(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """A^{-1} B via LU with partial pivoting."""
    A = np.asarray(A)
    B = np.asarray(B)
    if A.ndim != 2 or A.shape[0] != A.shape[1] or B.shape[0] != A.shape[0]:
        raise ValueError("dense_solve: dimension mismatch")
    lu, piv = sla.lu_factor(A, check_finite=True)
    if np.min(np.abs(np.diag(lu))) == 0.0:
        raise DecompositionFailure("dense_solve: singular pivot")
    return sla.lu_solve((lu, piv), B)


def form_temporal_core(M_t: np.ndarray, B_t: np.ndarray) -> np.ndarray:
    """C = (i B_t)^{-1} M_t = -i B_t^{-1} M_t."""
    M_t = np.asarray(M_t, dtype=float)
    B_t = np.asarray(B_t, dtype=float)
    lu, piv = sla.lu_factor(B_t)
    if np.min(np.abs(np.diag(lu))) < 1e-14 * max(np.linalg.norm(B_t), 1e-300):
        raise DecompositionFailure("temporal core: B_t is singular")
    return -1j * sla.lu_solve((lu, piv), M_t)


def spectral_condition(X: np.ndarray) -> float:
    """sigma_max / sigma_min; +inf if exactly singular."""
    s = sla.svdvals(X)
    return float("inf") if s[-1] == 0.0 else float(s[0] / s[-1])


def _normalise(w: np.ndarray, V: np.ndarray):
    V = V / np.linalg.norm(V, axis=0, keepdims=True)
    first = np.argmax(np.abs(V) > 0, axis=0)
    lead = V[first, np.arange(V.shape[1])]
    V = V * (np.abs(lead) / lead)[None, :]
    order = np.lexsort((w.imag, w.real))
    return w[order], V[:, order]


def eigen_decompose(A: np.ndarray, B_t: np.ndarray | None = None) -> TemporalFactors:
    """Eigendecomposition of the temporal core A = (iB_t)^{-1} M_t.

    `B_t` is needed for Y = X^{-1}(iB_t)^{-1}; without it Y = X^{-1}."""
    A = np.asarray(A, dtype=complex)
    if not np.isfinite(A).all():
        raise DecompositionFailure("eigen_decompose: non-finite entries")
    try:
        w, V = sla.eig(A)
    except sla.LinAlgError as exc:  # pragma: no cover
        raise DecompositionFailure(f"eigenvalue iteration did not converge: {exc}") from exc
    w, X = _normalise(w, V)
    s = sla.svdvals(X)
    if s[-1] < 1e-12:
        raise NotDiagonalizable(f"not diagonalizable: sigma_min(X) = {s[-1]:.3e} < 1e-12")
    rhs = np.eye(len(w), dtype=complex) if B_t is None else np.linalg.inv(1j * np.asarray(B_t, float))
    Y = dense_solve(X, rhs)
    return TemporalFactors(X=X, S=np.diag(w), Y=Y, kappa2=float(s[0] / s[-1]))


def schur_decompose(A: np.ndarray, B_t: np.ndarray | None = None) -> TemporalFactors:
    """Complex Schur form of the temporal core A = X S X^H:
    X unitary, S upper triangular with the eigenvalues on its diagonal,
    Y = X^H (iB_t)^{-1} (unitarity makes the inverse the conjugate transpose),
    kappa2 = 1.  The Bartels-Stewart variant's decomposition."""
    A = np.asarray(A, dtype=complex)
    if not np.isfinite(A).all():
        raise DecompositionFailure("schur_decompose: non-finite entries")
    try:
        S, X = sla.schur(A, output="complex")
    except sla.LinAlgError as exc:  # pragma: no cover
        raise DecompositionFailure(f"Schur iteration did not converge: {exc}") from exc
    n = A.shape[0]
    eps_dec = 1e-10 * n
    na = max(np.linalg.norm(A), 1e-300)
    if np.linalg.norm(A - X @ S @ X.conj().T) > eps_dec * na:
        raise DecompositionFailure("schur_decompose: residual above 1e-10 n_t ||A||")
    XH = X.conj().T
    Y = XH if B_t is None else XH @ np.linalg.inv(1j * np.asarray(B_t, float))
    return TemporalFactors(X=X, S=np.triu(S), Y=Y, kappa2=1.0, variant="schur")


def schur_factors(M_t: np.ndarray, B_t: np.ndarray) -> TemporalFactors:
    """Step 1 of the Bartels-Stewart solve: core and its complex Schur form."""
    return schur_decompose(form_temporal_core(M_t, B_t), B_t)


def temporal_factors(M_t: np.ndarray, B_t: np.ndarray) -> TemporalFactors:
    """Step 1 of the FD solve: core, eigendecomposition, Y, kappa_2."""
    return eigen_decompose(form_temporal_core(M_t, B_t), B_t)
