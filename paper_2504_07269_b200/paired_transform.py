"""Eigenpair-paired time transforms (K3p): the two FD transforms at half the flops.

The temporal pencil is real (M_t, B_t real), so the core
C = (i B_t)^{-1} M_t satisfies conj(C) = -C and its eigenvalues come in pairs
(lam, -conj(lam)) with eigenvectors x_p = c conj(x_l) (SURVEY.md Appendix A:
"Eigenvalues come in pairs (lam, -conj(lam))").  Consequently the rows of
Y = X^{-1} (i B_t)^{-1} pair as y_p = s conj(y_l).  The FD transforms of
SPEC.md:377 (G = Y F, Psi = X W) then need only the REAL and IMAGINARY parts
of one eigenvector per pair:

  forward:  with y_l = c + i d (real rows c, d), u = c F, v = d F:
            G_l = u + i v,   G_p = s (u - i v)
  back:     with x_l = a + i b, W'_l = W_l + c W_p, W'_p = i (W_l - c W_p):
            Psi = sum_l a W'_l + b W'_p           (a real x complex GEMM)

Both are real (n_t x n_t) x complex (n_t x N) GEMMs: 4 n_t^2 N real flops
instead of the 8 n_t^2 N of the complex product.  A self-paired eigenvalue
(lam = -conj(lam), purely imaginary) has x_l = e^{i phi} r with r real.

The pairing is verified numerically on the host (every rebuilt partner within
PAIR_TOL relative of LAPACK's); if any check fails the solver keeps the complex kernel
(`time_transform`) - a GPU kernel either way, no CPU path.

Host layout handed to the C-ABI (stfem_transform_pair_fwd / _back):
  * (both A matrices go to the device in the fragment-packed layout of
    pack_fragments: per 16-row block and k, the (row g, row g + 8) pairs)
  * A_fwd: (16 ceil(nsrc / 8), n_t) float64; block q of 16 rows holds
    Re y of sources 8q..8q+7 in rows 0-7 and Im y in rows 8-15, so one DMMA
    accumulator fragment holds c F and d F of the same source;
  * rows_fwd: int32 (nsrc, 2) = (l, p or -1), scale_fwd: complex (nsrc,) = s;
  * A_back: (n_t, n_t) float64, column l = Re x_l (or r), column p = Im x_l;
  * mix rows (npair, 2) and coefficients (npair, 4) complex of the in-place
    pre-pass [W_l; W_p] <- [[m00, m01], [m10, m11]] [W_l; W_p].
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

PAIR_TOL = 1e-7   # a rebuilt partner may move by the host eig's own error (3.5e-11 at n_t = 1024)


@dataclass
class PairedFactors:
    lam: np.ndarray          # (nt,) complex: lam_p = -conj(lam_l) exactly
    X: np.ndarray            # (nt, nt) complex: x_p = c conj(x_l) exactly
    Y: np.ndarray            # (nt, nt) complex: X^{-1} (i B_t)^{-1}, y_p = s conj(y_l) exactly
    A_fwd: np.ndarray        # (Mf, nt) float64
    rows_fwd: np.ndarray     # (nsrc, 2) int32
    scale_fwd: np.ndarray    # (nsrc,) complex128
    A_back: np.ndarray       # (nt, nt) float64
    mix_rows: np.ndarray     # (nmix, 2) int32 (p = -1: self-paired, only m00 applies)
    mix_coef: np.ndarray     # (nmix, 4) complex128
    npairs: int
    nself: int
    max_err: float           # largest relative change of a rebuilt partner eigenvector


def _match(lam: np.ndarray) -> list[tuple[int, int]] | None:
    """(l, p) with lam_p ~ -conj(lam_l); p == l for self-paired ones.  None when
    a match is missing or ambiguous (the runner-up is not 100x farther)."""
    n = lam.shape[0]
    scale = max(1.0, float(np.abs(lam).max()))
    D = np.abs(-np.conj(lam)[:, None] - lam[None, :])   # D[l, p] = |lam_p + conj(lam_l)|
    used = np.zeros(n, bool)
    out = []
    for l in np.argsort(D.min(axis=1), kind="stable"):
        if used[l]:
            continue
        d = np.where(used, np.inf, D[l])
        order = np.argsort(d)
        p = int(order[0])
        if not np.isfinite(d[p]) or d[p] > 1e-8 * scale:
            return None
        if n > 1 and np.isfinite(d[order[1]]) and d[order[1]] < 100 * max(d[p], 1e-14 * scale):
            return None
        used[l] = used[p] = True
        out.append((int(l), p))
    return out


def _rel(a: np.ndarray, b: np.ndarray) -> float:
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(a), 1e-300))


def build(lam: np.ndarray, X: np.ndarray, B_t: np.ndarray, tol: float = PAIR_TOL) -> PairedFactors | None:
    """Paired FD factors from the host eigendecomposition (lam, X) of the core.

    The partner of every pair is rebuilt from its lead (x_p := c conj(x_l),
    lam_p := -conj(lam_l): an exact eigenpair of the real pencil whenever
    (lam_l, x_l) is), self-paired vectors are made phase x real, and
    Y = X^{-1} (i B_t)^{-1} is recomputed and its rows paired exactly
    (y_p = -conj(y_l) / c).  The FD solution X diag(.) Y f is invariant under
    this change of eigenbasis.  None when the spectrum does not pair (the
    relative change of a partner must stay <= tol)."""
    lam = np.asarray(lam, np.complex128).copy()
    X = np.asarray(X, np.complex128).copy()
    nt = lam.shape[0]
    if nt % 2 or X.shape != (nt, nt):
        return None
    pairs = _match(lam)
    if pairs is None:
        return None
    err = 0.0
    cs = {}
    for l, p in pairs:
        xl = X[:, l]
        if p != l:
            c = np.vdot(np.conj(xl), X[:, p]) / np.vdot(xl, xl)
            newp = c * np.conj(xl)
            err = max(err, _rel(X[:, p], newp))
            X[:, p] = newp
            lam[p] = -np.conj(lam[l])
            cs[l] = c
        else:
            z = np.sum(xl * xl)                                  # e^{2 i phi} |r|^2
            ph = np.sqrt(z / abs(z)) if abs(z) > 0 else 1.0 + 0j
            newl = ph * (xl / ph).real
            err = max(err, _rel(xl, newl))
            X[:, l] = newl
            lam[l] = 1j * lam[l].imag
            cs[l] = ph
    if err > tol:
        return None
    Y = np.linalg.solve(X, np.linalg.inv(1j * np.asarray(B_t, float)))
    srcs, scales, mixr, mixc = [], [], [], []
    A_back = np.zeros((nt, nt))
    for l, p in pairs:
        if p != l:
            c = cs[l]
            s = -1.0 / c                                         # y_p = s conj(y_l)
            yl = 0.5 * (Y[l] + np.conj(Y[p] / s))
            Y[l], Y[p] = yl, s * np.conj(yl)
            srcs.append((l, p))
            scales.append(s)
            A_back[:, l] = X[:, l].real
            A_back[:, p] = X[:, l].imag
            mixr.append((l, p))
            mixc.append((1.0, c, 1j, -1j * c))
        else:
            ph = cs[l]
            srcs.append((l, -1))
            scales.append(0.0)
            A_back[:, l] = (X[:, l] / ph).real
            mixr.append((l, -1))
            mixc.append((ph, 0.0, 0.0, 0.0))
    nsrc = len(srcs)
    nblk = -(-nsrc // 8)
    A_fwd = np.zeros((16 * nblk, nt))
    for s_, (l, _) in enumerate(srcs):
        q, g = divmod(s_, 8)
        A_fwd[16 * q + g] = Y[l].real
        A_fwd[16 * q + 8 + g] = Y[l].imag
    return PairedFactors(lam=lam, X=X, Y=Y, A_fwd=A_fwd,
                         rows_fwd=np.asarray(srcs, np.int32).reshape(-1, 2),
                         scale_fwd=np.asarray(scales, np.complex128), A_back=A_back,
                         mix_rows=np.asarray(mixr, np.int32).reshape(-1, 2),
                         mix_coef=np.asarray(mixc, np.complex128).reshape(-1, 4),
                         npairs=sum(1 for l, p in pairs if p != l),
                         nself=sum(1 for l, p in pairs if p == l), max_err=err)


def forward_host(pf: PairedFactors, F: np.ndarray) -> np.ndarray:
    """numpy statement of the forward kernel (test helper): G = Y F."""
    nt = F.shape[0]
    U = pf.A_fwd @ F
    G = np.zeros((nt,) + F.shape[1:], np.complex128)
    for s, (l, p) in enumerate(pf.rows_fwd):
        q, g = divmod(s, 8)
        u, v = U[16 * q + g], U[16 * q + 8 + g]
        G[l] = u + 1j * v
        if p >= 0:
            G[p] = pf.scale_fwd[s] * (u - 1j * v)
    return G


def back_host(pf: PairedFactors, W: np.ndarray) -> np.ndarray:
    """numpy statement of the pre-pass + back kernel (test helper): Psi = X W."""
    W = W.copy()
    for (l, p), (m00, m01, m10, m11) in zip(pf.mix_rows, pf.mix_coef):
        if p >= 0:
            wl, wp = W[l].copy(), W[p].copy()
            W[l] = m00 * wl + m01 * wp
            W[p] = m10 * wl + m11 * wp
        else:
            W[l] = m00 * W[l]
    return pf.A_back @ W


def pack_fragments(A: np.ndarray) -> np.ndarray:
    """The kernels' A layout: P[mb, k, g, h] = A[16 mb + g + 8 h, k] (rows zero-padded to a
    multiple of 16), i.e. per 16-row block and k the 8 row pairs of one DMMA A fragment."""
    M, K = A.shape
    mb = -(-M // 16)
    Ap = np.zeros((16 * mb, K))
    Ap[:M] = A
    return np.ascontiguousarray(Ap.reshape(mb, 2, 8, K).transpose(0, 3, 2, 1))


class DevicePairs:
    """Device copies of a PairedFactors for the K3p kernels."""

    def __init__(self, pf: PairedFactors, device):
        import torch
        self.host = pf
        self.nt = pf.A_back.shape[0]
        self.A_fwd = torch.as_tensor(pack_fragments(pf.A_fwd), device=device)
        self.mrows_fwd = pf.A_fwd.shape[0]
        self.rows_fwd = torch.as_tensor(np.ascontiguousarray(pf.rows_fwd), device=device)
        self.scale_fwd = torch.as_tensor(np.ascontiguousarray(pf.scale_fwd), device=device)
        self.A_back = torch.as_tensor(pack_fragments(pf.A_back), device=device)
        self.mix_rows = torch.as_tensor(np.ascontiguousarray(pf.mix_rows), device=device)
        self.mix_coef = torch.as_tensor(np.ascontiguousarray(pf.mix_coef), device=device)
