"""Host setup of the spectral subtree elimination (csrc/spectral.cuh, K6).

Every shifted spatial system of the FD solve is K(lam) = M_x + lam A_x with
M_x, A_x real SPD and the same sparsity (one ordering for
all shifts :343).  The bottom subtrees of the nested-dissection tree are
therefore eliminated in closed form, once for all shifts: for a subtree with
interior DoFs I (all its pivots) and boundary Gam (its root's boundary rows),
the generalized eigendecomposition V^T A_II V = I, V^T M_II V = diag(theta)
gives

    K_II(lam)^{-1} = V diag(1 / (theta + lam)) V^T
    U(lam) = -K_GI K_II^{-1} K_IG = -(R diag(w) R^T + C0 + lam C1)

with P = M_GI V, Q = A_GI V, R = P - Q diag(theta), C1 = Q Q^T,
C0 = R Q^T + Q R^T + Q diag(theta) Q^T, w = 1 / (theta + lam).  The device
turns U, the forward RHS and the backward solve of every subtree into DMMA
GEMMs over the shifts; this module computes (V, theta, R, Q, C0, C1) per
subtree in fp64 on the host (LAPACK via numpy, batched by subtree size over
a thread pool), a one-off per mesh like the temporal eigendecomposition, and
hands them to the plan through `stfem_plan_set_spectral`.

Subtree roots: fronts whose subtree interior has at most `max_interior`
DoFs while their parent's has more (or no parent).
"""

from __future__ import annotations

import ctypes as C
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import scipy.sparse as sp

from . import _native as N

DEFAULT_MAX_INTERIOR = 256   # measured on C4 (ms/step): 200 -> 874, 256 -> 807, 320 -> 807


def subtree_first(fronts: np.ndarray) -> np.ndarray:
    """First pivot of every front's subtree (fronts in postorder: pbeg, p, n, parent, depth)."""
    first = fronts[:, 0].copy()
    for f in range(len(fronts)):
        par = fronts[f, 3]
        if par >= 0 and first[f] < first[par]:
            first[par] = first[f]
    return first


def select_roots(fronts: np.ndarray, max_interior: int) -> tuple[np.ndarray, np.ndarray]:
    first = subtree_first(fronts)
    m = fronts[:, 0] + fronts[:, 1] - first
    par = fronts[:, 3]
    ok = m <= max_interior
    parent_big = np.where(par >= 0, ~ok[np.maximum(par, 0)], True)
    roots = np.nonzero(ok & parent_big)[0].astype(np.int32)
    return roots, first[roots].astype(np.int32)


def _gen_eig(Ms: np.ndarray, As: np.ndarray):
    """Batched V^T A V = I, V^T M V = diag(theta) via Cholesky of A."""
    L = np.linalg.cholesky(As)
    Li = np.linalg.inv(L)
    Ct = Li @ Ms @ np.swapaxes(Li, -1, -2)
    Ct = 0.5 * (Ct + np.swapaxes(Ct, -1, -2))
    th, Wv = np.linalg.eigh(Ct)
    return th, np.swapaxes(Li, -1, -2) @ Wv


class SpectralData:
    """Packed per-subtree arrays in the layout stfem_plan_set_spectral expects."""

    def __init__(self, roots, first, offsets, V, theta, RQ, C01, m, g):
        self.roots, self.first, self.offsets = roots, first, offsets
        self.V, self.theta, self.RQ, self.C01 = V, theta, RQ, C01
        self.m, self.g = m, g

    @property
    def nroots(self) -> int:
        return len(self.roots)

    def nbytes(self) -> int:
        return 8 * (self.V.size + self.theta.size + self.RQ.size + self.C01.size)


def _signature(Mp, Ap, a: int, b: int, gam: np.ndarray, scale_m: float, scale_a: float):
    """Hashable signature of a subtree's (M_II, A_II, M_GI, A_GI): rows [a, b) of the permuted
    operators (their columns are the interior [a, b) and boundary rows, all numbered later), with
    interior columns relative to a, boundary columns as positions in `gam`, and the values rounded
    at 2^-36 of the operator's largest entry.  Subtrees of a (locally) uniform mesh that are
    translates of each other share it; anything else differs."""
    lo, hi = Mp.indptr[a], Mp.indptr[b]
    cols = Mp.indices[lo:hi].astype(np.int64)
    inside = cols < b
    rel = np.where(inside, cols - a, (b - a) + np.searchsorted(gam, cols))
    q = 2.0 ** 36
    return (b - a, len(gam), (Mp.indptr[a:b + 1] - lo).tobytes(), rel.tobytes(),
            np.round(Mp.data[lo:hi] * (q / scale_m)).astype(np.int64).tobytes(),
            np.round(Ap.data[lo:hi] * (q / scale_a)).astype(np.int64).tobytes())


def build(fronts: np.ndarray, front_rows, perm: np.ndarray, M_x: sp.spmatrix, A_x: sp.spmatrix,
          max_interior: int = DEFAULT_MAX_INTERIOR, threads: int | None = None,
          dedup: bool = True) -> SpectralData:
    """Spectral data of the plan's bottom subtrees (M_x, A_x in the original numbering).

    dedup: congruent subtrees -- same local pattern and the same M / A entries to 2^-36 relative,
    i.e. translates of one another on a uniform mesh (C4: 1024 subtrees in 20 classes; C5: 1021 in
    72) -- share ONE eigendecomposition and one copy of (V, theta, R, Q, C0, C1): the host setup
    and the device footprint shrink by the class ratio (C4: 0.8 GB -> 16 MB, which then lives in
    L2), at the price of representing a subtree by a class mate whose entries differ in the last
    bits (a relative perturbation <= 2^-36 of entries that are themselves rounded sums)."""
    roots, first = select_roots(fronts, max_interior)
    perm = np.asarray(perm, dtype=np.int64)
    Mp = sp.csr_matrix(M_x)[perm][:, perm].tocsr()
    Ap = sp.csr_matrix(A_x)[perm][:, perm].tocsr()
    Mp.sort_indices()
    Ap.sort_indices()
    same_pattern = np.array_equal(Mp.indptr, Ap.indptr) and np.array_equal(Mp.indices, Ap.indices)
    nr = len(roots)
    m = (fronts[roots, 0] + fronts[roots, 1] - first).astype(np.int64)
    g = (fronts[roots, 2] - fronts[roots, 1]).astype(np.int64)
    gams = [np.asarray(front_rows[roots[t]][fronts[roots[t], 1]:], dtype=np.int64) for t in range(nr)]
    # classes of congruent subtrees: rep[c] = representative subtree, cls[t] = class of subtree t
    cls = np.arange(nr)
    rep = list(range(nr))
    if dedup and same_pattern and nr:
        sm_, sa_ = float(np.abs(Mp.data).max()), float(np.abs(Ap.data).max())
        seen, rep = {}, []
        for t in range(nr):
            key = _signature(Mp, Ap, int(first[t]), int(first[t] + m[t]), gams[t], sm_, sa_)
            c = seen.get(key)
            if c is None:
                c = seen[key] = len(rep)
                rep.append(t)
            cls[t] = c
    rep = np.asarray(rep, dtype=np.int64)
    nc = len(rep)
    mc, gc = m[rep], g[rep]
    coffs = np.zeros((nc, 4), dtype=np.int64)
    if nc:
        coffs[1:, 0] = np.cumsum(mc * mc)[:-1]
        coffs[1:, 1] = np.cumsum(mc)[:-1]
        coffs[1:, 2] = np.cumsum(2 * gc * mc)[:-1]
        coffs[1:, 3] = np.cumsum(2 * gc * gc)[:-1]
    V = np.zeros(int((mc * mc).sum()))
    theta = np.zeros(int(mc.sum()))
    RQ = np.zeros(int((2 * gc * mc).sum()))
    C01 = np.zeros(int((2 * gc * gc).sum()))

    def blocks(t):
        a, b = int(first[t]), int(first[t] + m[t])
        gam = gams[t]
        return (Mp[a:b, a:b].toarray(), Ap[a:b, a:b].toarray(), Mp[gam][:, a:b].toarray(),
                Ap[gam][:, a:b].toarray())

    def work(cs):
        Ms, As, MG, AG = zip(*(blocks(int(rep[c])) for c in cs))
        th, Vb = _gen_eig(np.stack(Ms), np.stack(As))
        for q, c in enumerate(cs):
            mt, gt = int(mc[c]), int(gc[c])
            Vt, tt = Vb[q], th[q]
            P = MG[q] @ Vt
            Q = AG[q] @ Vt
            R = P - Q * tt
            C1 = Q @ Q.T
            C0 = R @ Q.T + Q @ R.T + (Q * tt) @ Q.T
            V[coffs[c, 0]:coffs[c, 0] + mt * mt] = Vt.T.ravel()           # column-major V[i + k m]
            theta[coffs[c, 1]:coffs[c, 1] + mt] = tt
            RQ[coffs[c, 2]:coffs[c, 2] + gt * mt] = R.T.ravel()          # column-major R[i + k g]
            RQ[coffs[c, 2] + gt * mt:coffs[c, 2] + 2 * gt * mt] = Q.T.ravel()
            C01[coffs[c, 3]:coffs[c, 3] + gt * gt] = C0.T.ravel()
            C01[coffs[c, 3] + gt * gt:coffs[c, 3] + 2 * gt * gt] = C1.T.ravel()

    # batches of equal interior size (batched LAPACK), spread over host threads
    chunks = []
    for mv in np.unique(mc):
        cs = np.nonzero(mc == mv)[0]
        step = max(1, min(64, (len(cs) + 7) // 8))
        chunks += [cs[i:i + step] for i in range(0, len(cs), step)]
    nth = threads or len(os.sched_getaffinity(0))
    if int((mc ** 3).sum()) < 2 * 10 ** 9 or nth <= 1:
        # a few classes of congruent subtrees (C4: 20 x 225^3): serial, no BLAS pinning -- a
        # process-wide thread limit here would starve a concurrent temporal eigendecomposition
        for cs in chunks:
            work(cs)
    else:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1), ThreadPoolExecutor(max(1, nth)) as ex:
            list(ex.map(work, chunks))
    offs = coffs[cls] if nr else np.zeros((0, 4), dtype=np.int64)      # every subtree points at its class data
    data = SpectralData(roots, first, np.ascontiguousarray(offs).ravel().copy(), V, theta, RQ, C01, m, g)
    data.classes, data.cls = nc, cls
    return data


def attach(plan_handle, data: SpectralData | None):
    """stfem_plan_set_spectral (data None or empty = plain multifrontal)."""
    lib = N.lib()
    if data is None or data.nroots == 0:
        N.check(lib.stfem_plan_set_spectral(plan_handle, 0, None, None, None, None, 0, None, 0, None, 0,
                                            None, 0))
        return
    arrs = [np.ascontiguousarray(x) for x in (data.roots.astype(np.int32), data.first.astype(np.int32),
                                              data.offsets.astype(np.int64))]
    vals = [np.ascontiguousarray(x, dtype=np.float64) for x in (data.V, data.theta, data.RQ, data.C01)]
    N.check(lib.stfem_plan_set_spectral(
        plan_handle, data.nroots, arrs[0].ctypes.data, arrs[1].ctypes.data, arrs[2].ctypes.data,
        vals[0].ctypes.data, vals[0].size, vals[1].ctypes.data, vals[1].size, vals[2].ctypes.data,
        vals[2].size, vals[3].ctypes.data, vals[3].size))


def stats(plan_handle) -> dict:
    nr = C.c_int32()
    fu, fr = C.c_double(), C.c_double()
    nb = C.c_int64()
    N.check(N.lib().stfem_plan_spectral_stats(plan_handle, C.byref(nr), C.byref(fu), C.byref(fr), C.byref(nb)))
    return {"nroots": nr.value, "flops_u": fu.value, "flops_rhs": fr.value, "bytes": nb.value}
