"""Batched sparse direct solver for the shifted spatial systems.

`SpatialPlan` = one host symbolic analysis per sparsity pattern (geometric
nested dissection, supernodal tree, extend-add maps; csrc/symbolic.cpp),
shared by every shift.  The numeric multifrontal
complex-symmetric LDL^T factorization and both triangular solves run on the
GPU, batched across shifts (csrc/multifrontal.cu).

SPEC API: `factor(M_x, A_x, lam) -> SpatialFactorization`, `solve(fact, b)`.
Factors are never materialised for later reuse on the device (they are
streamed per batch of shifts, SURVEY.md §7 hard part 4), so a
`SpatialFactorization` records (plan, operators, shifts) and `solve` runs the
fused factor + solve.  `factor_solve_batch` is the batched form used by the
FD solver.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import spectral as SP
from .fem_assembly import SpatialOperators


class SpatialPlan:
    """Symbolic analysis + device tables for one spatial pattern.

    spectral: max interior DoFs of the subtrees eliminated in closed form
    (K6, spectral.py); 0 = plain multifrontal; None = the default (256).  The
    spectral data depends on the operator values, so it is built from `ops`
    when they are assembled (here, or on the first factor_solve) and rebuilt
    when `ops.assemble()` produces new value tensors.

    options: stfem_plan_options fields to override (small_front_n, fused_min_p,
    panel_group, asm_whole_n, level_timing, tiles_per_cta, ws_stages, bwd_dmma_min_p,
    workspace_fraction, pivot_tol) -- the plan's only tuning interface (no environment
    variables)."""

    def __init__(self, ops: SpatialOperators, leaf_size: int = 16, spectral: int | None = None,
                 options: dict | None = None, spectral_threads: int | None = None):
        self.ops = ops
        self.n = ops.n
        h = C.c_void_p()
        N.check(N.lib().stfem_plan_create(ops.n, ops.rowptr.ctypes.data, ops.colind.ctypes.data,
                                          ops.coords.ctypes.data, 2, leaf_size, C.byref(h)))
        self._h = h
        st = N.plan_stats()
        N.check(N.lib().stfem_plan_stats_get(h, C.byref(st)))
        self.stats = {f: getattr(st, f) for f, _ in N.plan_stats._fields_}
        self.spectral_m = SP.DEFAULT_MAX_INTERIOR if spectral is None else int(spectral)
        self.spectral = None          # SpectralData once attached
        self.spectral_threads = spectral_threads
        self._spectral_key = None     # identity of the operator values the spectral data came from
        self.t_spectral = 0.0         # host setup seconds
        if options:
            self.set_options(**options)
        if self.spectral_m > 0 and ops.Mvals is not None:
            self._attach_spectral()

    def _ops_key(self):
        o = self.ops
        return (o.epoch, o.Mvals.data_ptr(), o.Avals.data_ptr(), o.Mvals._version, o.Avals._version)

    def options(self) -> dict:
        o = N.plan_options()
        N.check(N.lib().stfem_plan_get_options(self._h, C.byref(o)))
        return {f: getattr(o, f) for f, _ in N.plan_options._fields_}

    def set_options(self, **kw):
        o = N.plan_options()
        N.check(N.lib().stfem_plan_get_options(self._h, C.byref(o)))
        for k, v in kw.items():
            if k not in dict(N.plan_options._fields_):
                raise KeyError(f"unknown plan option {k!r}")
            setattr(o, k, v)
        N.check(N.lib().stfem_plan_set_options(self._h, C.byref(o)))

    def reserve(self, nshift: int, nrhs: int = 1):
        """Allocate the numeric workspace now (stfem_plan_reserve): later factor_solve calls
        of up to (nshift, nrhs) neither allocate nor synchronise the device."""
        N.require_cuda()
        if self.spectral_m > 0 and self.ops.Mvals is not None and self._spectral_key != self._ops_key():
            self._attach_spectral()
        N.check(N.lib().stfem_plan_reserve(self._h, int(nshift), int(min(nrhs, self.max_rhs()))))

    def prepare(self):
        """Bring the value-dependent plan data up to date with the operators (spectral subtree
        data are rebuilt when ops.assemble() produced new values) before a direct C-ABI call."""
        if self.ops.Mvals is None:
            raise RuntimeError("spatial operators are not assembled")
        if self.spectral_m > 0 and self._spectral_key != self._ops_key():
            self._attach_spectral()

    def max_rhs(self) -> int:
        mr = C.c_int32()
        N.check(N.lib().stfem_plan_max_rhs(self._h, C.byref(mr)))
        return max(1, mr.value)

    def check(self, stream=None):
        """stfem_plan_check: wait for the factor_solve calls issued on `stream` and raise
        SingularPivot (naming the shift) if one of them met a pivot collapse."""
        N.check(N.lib().stfem_plan_check(self._h, N.stream_ptr(stream)))

    def set_shift_base(self, base: int):
        N.check(N.lib().stfem_plan_set_shift_base(self._h, int(base)))

    def _attach_spectral(self):
        import time
        t0 = time.perf_counter()
        fr = self.fronts()
        data = SP.build(fr, self.front_rows(), self.perm(), self.ops.M_x.to_scipy(), self.ops.A_x.to_scipy(),
                        self.spectral_m, threads=self.spectral_threads)
        SP.attach(self._h, data)
        self.spectral = data
        self._spectral_key = self._ops_key()
        self.t_spectral = time.perf_counter() - t0
        st = N.plan_stats()
        N.check(N.lib().stfem_plan_stats_get(self._h, C.byref(st)))
        self.stats = {f: getattr(st, f) for f, _ in N.plan_stats._fields_}

    def spectral_stats(self) -> dict:
        return SP.stats(self._h)

    @property
    def handle(self):
        return self._h

    def perm(self) -> np.ndarray:
        p = np.empty(self.n, dtype=np.int32)
        N.check(N.lib().stfem_plan_perm(self._h, p.ctypes.data))
        return p

    def fronts(self) -> np.ndarray:
        t = np.empty((self.stats["num_fronts"], 5), dtype=np.int32)
        N.check(N.lib().stfem_plan_fronts(self._h, t.ctypes.data))
        return t

    def front_rows(self):
        """List of row-index arrays (new numbering) per front."""
        nf = self.stats["num_fronts"]
        off = np.empty(nf + 1, dtype=np.int64)
        N.check(N.lib().stfem_plan_front_rows(self._h, off.ctypes.data, None))
        rows = np.empty(off[-1], dtype=np.int32)
        N.check(N.lib().stfem_plan_front_rows(self._h, off.ctypes.data, rows.ctypes.data))
        return [rows[off[f]:off[f + 1]] for f in range(nf)]

    def record_levels(self, on: bool = True):
        N.check(N.lib().stfem_plan_record_levels(self._h, 1 if on else 0))

    def level_report(self):
        """(factor_ms[d], backward_ms[d], flops_per_shift[d], small[d]) of the last recorded call."""
        L = self.stats["depth"] + 1
        ms = np.zeros(2 * L)
        fl = np.zeros(L)
        sm = np.zeros(L, dtype=np.int32)
        N.check(N.lib().stfem_plan_level_report(self._h, ms.ctypes.data, fl.ctypes.data, sm.ctypes.data))
        return ms[:L], ms[L:], fl, sm.astype(bool)

    FAMILIES = ("spectral", "assembly", "diag", "trsm", "panel_update", "syrk", "backward", "small_factor")

    def kernel_report(self) -> dict:
        """{family: (ms of the last recorded call, algorithmic flops per shift, launches)}."""
        nf = len(self.FAMILIES)
        ms = np.zeros(nf)
        fl = np.zeros(nf)
        nl = np.zeros(nf, dtype=np.int64)
        N.check(N.lib().stfem_plan_kernel_report(self._h, nf, ms.ctypes.data, fl.ctypes.data, nl.ctypes.data))
        return {k: (float(ms[i]), float(fl[i]), int(nl[i])) for i, k in enumerate(self.FAMILIES)}

    def last_num_batches(self) -> int:
        """Shift batches used by the last factor_solve call."""
        v = C.c_int32()
        N.check(N.lib().stfem_plan_last_batches(self._h, C.byref(v)))
        return max(1, v.value)

    def last_launches(self) -> int:
        v = C.c_int64()
        N.check(N.lib().stfem_plan_last_launches(self._h, C.byref(v)))
        return v.value

    def set_batch(self, batch: int) -> int:
        bps = C.c_int64()
        N.check(N.lib().stfem_plan_set_batch(self._h, int(batch), C.byref(bps)))
        return bps.value

    def factor_solve(self, lam: torch.Tensor, G: torch.Tensor, W: torch.Tensor, layout: N.bv_layout,
                     nrhs: int, stream=None, check: bool = True, permuted: bool = False):
        """(M_x + lam[s] A_x) W[r, s] = G[r, s] for every shift s (device c128).

        The C call only enqueues work.  check=True (default) then waits for it and raises
        SingularPivot if a shift was numerically singular; pipelined
        callers pass check=False and call `plan.check()` once at the end."""
        N.require_cuda(G)
        ops = self.ops
        if ops.Mvals is None:
            raise RuntimeError("spatial operators are not assembled")
        if self.spectral_m > 0 and self._spectral_key != self._ops_key():
            self._attach_spectral()     # first use, or ops.assemble() produced new values
        lam = lam.to(device=G.device, dtype=torch.complex128).contiguous()
        # permuted: G and W are indexed in the plan's numbering (the FD solver's transforms apply
        # the permutation, kronecker_solver.FDMSolver._fwd_block / _back_block)
        N.check(N.lib().stfem_plan_set_io_permuted(self._h, 1 if permuted else 0))
        step = self.max_rhs()
        for r0 in range(0, nrhs, step):
            nr = min(step, nrhs - r0)
            off = r0 * layout.rhs_stride
            N.check(N.lib().stfem_factor_solve(
                self._h, N.ptr(ops.Mvals), N.ptr(ops.Avals), N.ptr(lam), lam.numel(), nr,
                C.c_void_p(G.data_ptr() + 16 * off), C.c_void_p(W.data_ptr() + 16 * off), layout,
                N.stream_ptr(stream)))
        if check:
            self.check(stream)
        return W

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and N is not None and N._lib is not None:
            N._lib.stfem_plan_destroy(h)
            self._h = None


def blockvector_layout(nt: int, nx: int) -> N.bv_layout:
    """Layout of a (n_rhs, n_t, n_x) stack of BlockVectors."""
    return N.bv_layout(nt * nx, nx, nx, 0)


@dataclass(frozen=True)
class SpatialFactorization:
    """K_lam = M_x + lam A_x over a shared plan."""

    plan: SpatialPlan
    lam: complex

    @property
    def n(self) -> int:
        return self.plan.n


def _same_operator(given, mine) -> bool:
    """Is `given` (SparseRealMatrix, scipy matrix or value tensor) the plan's operator?"""
    vals = getattr(given, "values", given)
    if torch.is_tensor(vals):
        return vals.data_ptr() == mine.values.data_ptr() or (
            vals.shape == mine.values.shape and bool(torch.equal(vals.to(mine.values.device), mine.values)))
    try:
        import scipy.sparse as sp
        g = sp.csr_matrix(given)
        g.sort_indices()
        m = mine.to_scipy()
        return g.shape == m.shape and np.array_equal(g.indptr, m.indptr) and np.array_equal(g.indices, m.indices) \
            and np.array_equal(g.data, m.data)
    except Exception:
        return False


def factor(plan_or_ops, M_x=None, A_x=None, lam: complex = 0j) -> SpatialFactorization:
    """SPEC.md:323-331.  `plan_or_ops` is a SpatialPlan (or SpatialOperators, for which a
    plan is built).  M_x / A_x, when given, must BE the plan's operators (same pattern and
    values): the factorization always uses the plan's device-resident values, so anything
    else raises DimensionMismatch instead of silently solving a different system.  The
    numeric factors are streamed inside `solve` (never kept), so a singular shift is
    reported there (SingularPivot)."""
    plan = plan_or_ops if isinstance(plan_or_ops, SpatialPlan) else SpatialPlan(plan_or_ops)
    for given, mine, name in ((M_x, "M_x", "M_x"), (A_x, "A_x", "A_x")):
        if given is None:
            continue
        if plan.ops.Mvals is None or not _same_operator(given, getattr(plan.ops, mine)):
            raise N.DimensionMismatch(N.ERR_DIM, f"factor: {name} is not the plan's operator (build a SpatialPlan "
                                                 "from the operators you want to factor)")
    return SpatialFactorization(plan, complex(lam))


def solve(fact: SpatialFactorization, b: torch.Tensor) -> torch.Tensor:
    """w with K_lam w = b (b: (n_x,) or (n_rhs, n_x) complex128 on the GPU)."""
    n = fact.n
    if b.shape[-1] != n:
        raise N.DimensionMismatch(N.ERR_DIM, f"solve: rhs length {b.shape[-1]} != n_x {n}")
    bb = b.reshape(-1, n).to(torch.complex128).contiguous()
    W = torch.empty_like(bb)
    lam = torch.tensor([fact.lam], dtype=torch.complex128, device=bb.device)
    fact.plan.factor_solve(lam, bb, W, N.bv_layout(n, 0, n, 0), bb.shape[0])
    return W.reshape(b.shape)


def factor_solve_batch(plan: SpatialPlan, lam, G: torch.Tensor, W: torch.Tensor | None = None):
    """W[r, l] = (M_x + lam_l A_x)^{-1} G[r, l] for G of shape (n_t, n_x) or (n_rhs, n_t, n_x)."""
    single = G.dim() == 2
    Gb = (G.unsqueeze(0) if single else G).contiguous()
    nr, nt, nx = Gb.shape
    if W is None:
        W = torch.empty_like(Gb)
    lam_t = torch.as_tensor(np.asarray(lam), dtype=torch.complex128, device=G.device)
    if lam_t.numel() != nt:
        raise N.DimensionMismatch(N.ERR_DIM, "factor_solve_batch: one shift per temporal block")
    plan.factor_solve(lam_t, Gb, W, blockvector_layout(nt, nx), nr)
    return W[0] if single else W
