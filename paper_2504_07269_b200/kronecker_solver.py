"""Kronecker space-time solver, fast-diagonalization variant.

  solve(ops, M_t, B_t, f, variant=FastDiagonalization) -> SolveReport
    (1) temporal core + eigendecomposition (host fp64, `t_setup`)
    (2) G = (Y (x) I) F                     K3p/K3 DMMA GEMM
    (3) (M_x + lam_l A_x) w_l = g_l         K4/K5 multifrontal SPEC.md:377, :415
    (4) Psi = (X (x) I) W                   K3p/K3 DMMA GEMM
  K3p (paired_transform.py) runs both transforms at half the flops of the
  complex GEMM K3 by pairing the eigenvalues (lam, -conj(lam)) of the real
  temporal pencil; K3 remains for factors that do not pair (and for BS).
  transform_blocks(T, v)   -> K3
  apply_global(...)   -> K7 (residual certificate, :405)

Kronecker factors are never materialised.  The Bartels-Stewart
variant (`BSSolver`) runs the same kernels with a
strictly sequential sweep; there is no silent fallback between the variants
(SPEC.md:412): a defective core raises `NotDiagonalizable` under FD.  All device work is stream-ordered; stage times are
CUDA-event times on the launching stream.
"""

from __future__ import annotations

import ctypes as C
import enum
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _kernels as K
from . import _native as N
from . import paired_transform as PT
from .dense_complex_linalg import TemporalFactors, temporal_factors
from .fem_assembly import SpatialOperators, temporal_band
from .sparse_spatial_solver import SpatialPlan, blockvector_layout

C128 = torch.complex128


class SolverVariant(enum.Enum):
    BartelsStewart = "bs"
    FastDiagonalization = "fd"


@dataclass
class SolveReport:
    """SPEC.md:364-371."""

    solution: torch.Tensor
    solve_seconds: float
    kappa2: float
    relative_residual: float | None
    timings: dict = field(default_factory=dict)


def transform_blocks(T, v: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """out_l = sum_k T[l,k] v_k for v of shape (n_t, n_x) or (n_rhs, n_t, n_x)."""
    Tt = torch.as_tensor(np.asarray(T) if not torch.is_tensor(T) else T, dtype=C128, device=v.device)
    return K.time_transform(Tt, v, out=out, stream=stream)


def apply_global(ops: SpatialOperators, M_t: np.ndarray, B_t: np.ndarray, v: torch.Tensor,
                 stream=None) -> torch.Tensor:
    """(i B_t (x) M_x + M_t (x) A_x) v, matrix-free (banded in time)."""
    nt = M_t.shape[0]
    if v.shape[-2:] != (nt, ops.n):
        raise N.DimensionMismatch(N.ERR_DIM, f"apply_global: v {tuple(v.shape)} vs ({nt}, {ops.n})")
    bw = 1 if np.count_nonzero(np.triu(M_t, 2)) == 0 and np.count_nonzero(np.triu(B_t, 2)) == 0 else 2
    Mb = torch.as_tensor(temporal_band(M_t, bw), device=v.device)
    Bb = torch.as_tensor(temporal_band(B_t, bw), device=v.device)
    vb = v.reshape(-1, nt, ops.n)
    out = torch.empty_like(vb)
    work = torch.empty((2, nt, ops.n), dtype=C128, device=v.device)
    for r in range(vb.shape[0]):
        vr = vb[r].contiguous()
        N.check(N.lib().stfem_apply_global(ops.handle, N.ptr(ops.Mvals), N.ptr(ops.Avals), N.ptr(Mb),
                                           N.ptr(Bb), bw, nt, N.ptr(vr), N.ptr(out[r]), N.ptr(work),
                                           N.stream_ptr(stream)))
    return out.reshape(v.shape)


def relative_residual(ops, M_t, B_t, psi: torch.Tensor, f: torch.Tensor) -> float:
    """max over RHS of ||A psi - f|| / ||f||, one RHS at a time
    so the temporaries stay O(n_t n_x)."""
    fb = f.reshape(-1, *f.shape[-2:])
    pb = psi.reshape(-1, *psi.shape[-2:])
    worst = 0.0
    for i in range(fb.shape[0]):
        r = apply_global(ops, M_t, B_t, pb[i])
        r.sub_(fb[i])
        nf = float(torch.linalg.vector_norm(fb[i]))
        nr = float(torch.linalg.vector_norm(r))
        del r
        worst = max(worst, nr / nf if nf > 0 else nr)
    return worst


def _as_stack(buf: torch.Tensor, like: torch.Tensor, name: str) -> torch.Tensor:
    """View of a caller buffer as the (n_rhs, n_t, n_x) stack; never a silent copy."""
    if buf.dtype != like.dtype or buf.device != like.device or buf.numel() != like.numel() \
            or not buf.is_contiguous():
        raise ValueError(f"solve: `{name}` must be a contiguous complex128 device buffer of F's shape")
    return buf.view(like.shape)


class FDMSolver:
    """Reusable FD solver for one (spatial mesh, temporal mesh) pair.

    setup(): temporal eigendecomposition (host fp64) + symbolic analysis,
    uploaded once; solve(F): steps 2-4 on the GPU."""

    def __init__(self, ops: SpatialOperators, M_t: np.ndarray, B_t: np.ndarray,
                 plan: SpatialPlan | None = None, factors: TemporalFactors | None = None,
                 leaf_size: int = 16, paired: bool = True):
        t0 = time.perf_counter()
        self.ops = ops
        self.M_t = np.asarray(M_t, float)
        self.B_t = np.asarray(B_t, float)
        self.nt = self.M_t.shape[0]
        # (Running the temporal eigendecomposition on a worker thread beside the spatial setup was
        # measured twice and dropped: round 1, eig 1.7 -> 3.5 s because the spectral build pinned
        # BLAS to one thread process-wide; round 2, with that build serial and unpinned, zgeev
        # still slowed from 1.57 to 4.85 s (C4) and 10.6 s (C5) beside the symbolic analysis on
        # the 16-core host.)
        box = {}
        t = time.perf_counter()
        tf = factors if factors is not None else temporal_factors(self.M_t, self.B_t)
        box.update(tf=tf, pf=PT.build(tf.eigenvalues, tf.X, self.B_t) if paired else None)
        box["t"] = time.perf_counter() - t
        t1 = time.perf_counter()
        self.plan = plan if plan is not None else SpatialPlan(ops, leaf_size)
        t2 = time.perf_counter()
        self.tf = box["tf"]
        dev = ops.device
        lam, X, Y = self.tf.eigenvalues, self.tf.X, self.tf.Y
        self.pairs = None
        pf = box["pf"]
        if pf is not None:
            # the paired eigenbasis (partners rebuilt from their leads) drives every stage
            lam, X, Y = pf.lam, pf.X, pf.Y
            self.pairs = PT.DevicePairs(pf, dev)
        # row-major on the device: the C-ABI takes raw pointers (LAPACK hands back Fortran order)
        self.X = torch.as_tensor(np.ascontiguousarray(X), dtype=C128, device=dev).contiguous()
        self.Y = torch.as_tensor(np.ascontiguousarray(Y), dtype=C128, device=dev).contiguous()
        self.lam = torch.as_tensor(np.ascontiguousarray(lam), dtype=C128, device=dev).contiguous()
        self.t_eig = box["t"]
        self.t_symbolic = t2 - t1
        self.t_setup = time.perf_counter() - t0
        self._ffi = None

    @property
    def kappa2(self) -> float:
        return self.tf.kappa2

    def fd_factors(self) -> N.fd_factors:
        """stfem_fd_factors over this solver's device-resident temporal factors."""
        if self._ffi is None:
            f = N.fd_factors()
            f.nt = self.nt
            f.lam = self.lam.data_ptr()
            f.X, f.Y = self.X.data_ptr(), self.Y.data_ptr()
            if self.pairs is not None:
                p = self.pairs
                f.A_fwd, f.mrows_fwd = p.A_fwd.data_ptr(), p.mrows_fwd
                f.rows_fwd, f.scale_fwd, f.nsrc = p.rows_fwd.data_ptr(), p.scale_fwd.data_ptr(), p.rows_fwd.shape[0]
                f.A_back = p.A_back.data_ptr()
                f.mix_rows, f.mix_coef, f.nmix = p.mix_rows.data_ptr(), p.mix_coef.data_ptr(), p.mix_rows.shape[0]
            self._ffi = f
        return self._ffi

    def forward_transform(self, F: torch.Tensor, out: torch.Tensor, stream=None) -> torch.Tensor:
        """G = (Y (x) I) F (step 2): K3p when the eigenvalues pair, else K3."""
        if self.pairs is not None:
            return K.transform_pair_fwd(self.pairs, F, out=out, stream=stream)
        return K.time_transform(self.Y, F, out=out, stream=stream)

    def back_transform(self, W: torch.Tensor, out: torch.Tensor, stream=None) -> torch.Tensor:
        """Psi = (X (x) I) W (step 4).  W is scratch: K3p mixes its pair rows in place."""
        if self.pairs is not None:
            return K.transform_pair_back(self.pairs, W, out=out, stream=stream)
        return K.time_transform(self.X, W, out=out, stream=stream)

    # ---- the spatial permutation fused into the transforms (paired transforms only; opt-in) ----
    # With fused_perm the forward transform scatters its result columns to the plan's numbering
    # (column iperm[x]) and the back transform gathers its operand columns from there, so the
    # spatial solves in between read G and write W with contiguous pivot rows
    # (stfem_plan_set_io_permuted) and no kernel gathers through the permutation.  Measured A/B
    # (tools/ab_fused.py, ms per solve, fused / not): C4 576.6 / 575.0, C5 1299.4 / 1293.3 -- the
    # solves gain 1-2 ms, the gathering back transform (16-byte cp.async per element instead of
    # bulk-copied tiles) loses 3: off by default.
    fused_perm = False

    @property
    def _fused(self) -> bool:
        return bool(self.fused_perm) and self.pairs is not None   # the column maps exist on K3p only

    def _iperm(self) -> torch.Tensor:
        if getattr(self, "_iperm_d", None) is None:
            perm = self.plan.perm()
            ip = np.empty_like(perm)
            ip[perm] = np.arange(len(perm), dtype=perm.dtype)
            self._iperm_d = torch.as_tensor(ip.astype(np.int32), device=self.X.device)
        return self._iperm_d

    def _fwd_block(self, Fblk: torch.Tensor, G: torch.Tensor, c0: int, c1: int, stream=None):
        """Forward transform of spatial columns [c0, c1) (Fblk) into the whole stack G."""
        if self._fused:
            return K.transform_pair_fwd(self.pairs, Fblk, out=G, stream=stream, out_cols=self._iperm()[c0:c1])
        return self.forward_transform(Fblk, G[..., c0:c1], stream)

    def _back_block(self, W: torch.Tensor, out_blk: torch.Tensor, c0: int, c1: int, stream=None):
        """Back transform into spatial columns [c0, c1) (out_blk) from the whole stack W (fused:
        `K.pair_mix` must have run over W)."""
        if self._fused:
            return K.transform_pair_back(self.pairs, W, out=out_blk, stream=stream, in_cols=self._iperm()[c0:c1],
                                         mixed=True)
        return self.back_transform(W[..., c0:c1], out_blk, stream)

    def _spatial_solves(self, G, W, nr, stream):
        self.plan.factor_solve(self.lam, G, W, blockvector_layout(self.nt, self.ops.n), nr, stream=stream,
                               check=False, permuted=self._fused)
        if self._fused:
            K.pair_mix(self.pairs, W, stream=stream)

    def solve(self, F: torch.Tensor, out: torch.Tensor | None = None, work: torch.Tensor | None = None,
              stream=None, timings: dict | None = None, check: bool = True) -> torch.Tensor:
        """Psi for F of shape (n_t, n_x) or (n_rhs, n_t, n_x), complex128 on the GPU.
        `out` / `work` (if given) must be contiguous buffers of F's shape, distinct from F
        and from each other; `work` is scratch.  check=False leaves the stream un-waited
        (stream-ordered pipelines); the caller then runs `self.plan.check()` itself."""
        N.require_cuda(F)
        if F.shape[-2:] != (self.nt, self.ops.n):
            raise N.DimensionMismatch(N.ERR_DIM, f"solve: f {tuple(F.shape)} vs ({self.nt}, {self.ops.n})")
        single = F.dim() == 2
        Fb = (F.unsqueeze(0) if single else F).contiguous()
        nr = Fb.shape[0]
        # buffer rotation without copies: F -> G (=out) -> W (=work) -> out
        G = _as_stack(out, Fb, "out") if out is not None else torch.empty_like(Fb)
        W = _as_stack(work, Fb, "work") if work is not None else torch.empty_like(Fb)
        if len({Fb.data_ptr(), G.data_ptr(), W.data_ptr()}) != 3:
            raise ValueError("solve: F, out and work must be three distinct buffers")
        s = stream if stream is not None else torch.cuda.current_stream()
        if timings is None:
            # the product path: steps 2-4 behind ONE C-ABI call (stfem_fdm_solve); the staged
            # path below runs the same three entry points with CUDA events in between
            self.plan.prepare()
            N.check(N.lib().stfem_fdm_solve(self.plan.handle, None, N.ptr(self.ops.Mvals), N.ptr(self.ops.Avals),
                                            C.byref(self.fd_factors()), N.ptr(Fb), N.ptr(G), N.ptr(W), nr,
                                            N.stream_ptr(s)))
            if check:
                self.plan.check(s)
            if out is not None:
                return out
            return G[0] if single else G
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if timings is not None else None
        if ev:
            ev[0].record(s)
        nx = self.ops.n
        self._fwd_block(Fb, G, 0, nx, s)                               # (2)
        if ev:
            ev[1].record(s)
        self._spatial_solves(G, W, nr, s)                              # (3) (+ the pair pre-pass of step 4)
        if ev:
            ev[2].record(s)
        self._back_block(W, G, 0, nx, s)                               # (4) (W is scratch)
        if check:
            self.plan.check(s)       # SingularPivot names the shift; waits for the stream
        if ev:
            ev[3].record(s)
            ev[3].synchronize()
            timings["forward_transform_s"] = ev[0].elapsed_time(ev[1]) / 1e3
            timings["factor_solve_s"] = ev[1].elapsed_time(ev[2]) / 1e3
            timings["back_transform_s"] = ev[2].elapsed_time(ev[3]) / 1e3
        if out is not None:
            return out
        return G[0] if single else G


    def solve_host(self, F_host: torch.Tensor, out_host: torch.Tensor, chunks: int = 8, stream=None,
                   dev_buffers: tuple | None = None) -> torch.Tensor:
        """Psi for a PINNED host F (n_rhs, n_t, n_x) into pinned host `out_host`.

        The host->device copy of spatial column block c+1 overlaps the forward
        transform of block c (each output column needs only its own input
        column), and the device->host copy of block c overlaps the back
        transform of block c+1; the spatial solves need every column and run
        in between.  `dev_buffers` = (F_d, G, W) reuses device storage."""
        N.require_cuda()
        Fh = F_host.unsqueeze(0) if F_host.dim() == 2 else F_host
        Ph = out_host.unsqueeze(0) if out_host.dim() == 2 else out_host
        if Fh.shape[-2:] != (self.nt, self.ops.n) or Ph.shape != Fh.shape:
            raise N.DimensionMismatch(N.ERR_DIM, f"solve_host: f {tuple(F_host.shape)} vs ({self.nt}, {self.ops.n})")
        if not (Fh.is_pinned() and Ph.is_pinned() and Fh.is_contiguous() and Ph.is_contiguous()):
            raise ValueError("solve_host: host buffers must be contiguous pinned memory")
        nr, nt, nx = Fh.shape
        dev = self.X.device
        if dev_buffers is None:
            dev_buffers = tuple(torch.empty(Fh.shape, dtype=C128, device=dev) for _ in range(3))
        Fd, G, W = dev_buffers[:3]
        s = stream if stream is not None else torch.cuda.current_stream()
        if getattr(self, "_copy_stream", None) is None:
            self._copy_stream = torch.cuda.Stream(device=dev)
        cs = self._copy_stream
        lib = N.lib()
        cw = -(-nx // max(1, chunks))
        blocks = [(c0, min(nx, c0 + cw)) for c0 in range(0, nx, cw)]
        start = torch.cuda.Event()
        start.record(s)
        cs.wait_event(start)
        for c0, c1 in blocks:                                             # (2) pipelined with H2D
            N.check(lib.stfem_copy_cols(N.ptr(Fd[..., c0:]), nx, C.c_void_p(Fh.data_ptr() + 16 * c0), nx,
                                        c1 - c0, nr * nt, 0, N.stream_ptr(cs)))
            ev = torch.cuda.Event()
            ev.record(cs)
            s.wait_event(ev)
            self._fwd_block(Fd[..., c0:c1], G, c0, c1, s)
        self._spatial_solves(G, W, nr, s)                                 # (3)
        for c0, c1 in blocks:                                             # (4) pipelined with D2H
            self._back_block(W, G[..., c0:c1], c0, c1, s)
            ev = torch.cuda.Event()
            ev.record(s)
            cs.wait_event(ev)
            N.check(lib.stfem_copy_cols(C.c_void_p(Ph.data_ptr() + 16 * c0), nx, N.ptr(G[..., c0:]), nx,
                                        c1 - c0, nr * nt, 1, N.stream_ptr(cs)))
        done = torch.cuda.Event()
        done.record(cs)
        s.wait_event(done)
        self.plan.check(s)
        return out_host


    def solve_host_stream(self, F_hosts, out_hosts, chunks: int = 8, stream=None,
                          dev_buffers: tuple | None = None):
        """Psi_k for a sequence of PINNED host RHS stacks F_hosts[k] into out_hosts[k]
        (streamed solves, e.g. a serving loop): every step still copies its F in and its
        Psi out, but step k+1's host->device copy runs on its own copy stream during
        step k's spatial solves, and step k's device->host copy (column blocks, behind
        the back transform) during step k+1's forward transform.  Three device buffers
        rotate: A holds the uploaded F; G and W swap roles every step (G_k = W_{k-1}:
        the buffer of Psi_{k-1} is only rewritten by factor_solve(k+1) once its copy has
        drained).  Returns out_hosts."""
        N.require_cuda()
        n = len(F_hosts)
        if n == 0:
            return out_hosts
        Fh = [f.unsqueeze(0) if f.dim() == 2 else f for f in F_hosts]
        Ph = [o.unsqueeze(0) if o.dim() == 2 else o for o in out_hosts]
        shape = Fh[0].shape
        for f, o in zip(Fh, Ph):
            if f.shape != shape or o.shape != shape or f.shape[-2:] != (self.nt, self.ops.n):
                raise N.DimensionMismatch(N.ERR_DIM, f"solve_host_stream: f {tuple(f.shape)} vs ({self.nt}, {self.ops.n})")
            if not (f.is_pinned() and o.is_pinned() and f.is_contiguous() and o.is_contiguous()):
                raise ValueError("solve_host_stream: host buffers must be contiguous pinned memory")
        nr, nt, nx = shape
        dev = self.X.device
        if dev_buffers is None:
            # a fourth buffer (when four stacks are a small part of the device memory) lets Psi_k
            # drain to the host during the whole of step k + 1 instead of having to be gone before
            # factor_solve(k + 1) overwrites it
            nbytes = 16 * nr * nt * nx
            total = torch.cuda.get_device_properties(dev).total_memory
            dev_buffers = tuple(torch.empty(shape, dtype=C128, device=dev) for _ in range(4 if 4 * nbytes <= 0.2 * total else 3))
        A = dev_buffers[0]
        four = len(dev_buffers) >= 4
        s = stream if stream is not None else torch.cuda.current_stream()
        if getattr(self, "_h2d_stream", None) is None:
            self._h2d_stream = torch.cuda.Stream(device=dev)
            self._d2h_stream = torch.cuda.Stream(device=dev)
        hs, ds = self._h2d_stream, self._d2h_stream
        lib = N.lib()
        cw = -(-nx // max(1, chunks))
        blocks = [(c0, min(nx, c0 + cw)) for c0 in range(0, nx, cw)]
        layout = blockvector_layout(nt, nx)

        def h2d(k, c0, c1):
            N.check(lib.stfem_copy_cols(N.ptr(A[..., c0:]), nx, C.c_void_p(Fh[k].data_ptr() + 16 * c0), nx,
                                        c1 - c0, nr * nt, 0, N.stream_ptr(hs)))

        start = torch.cuda.Event()
        start.record(s)
        hs.wait_event(start)
        ds.wait_event(start)
        d2h_done = None
        d2h_events = []
        for k in range(n):
            if four:   # W fixed; G (which also receives Psi_k) alternates: Psi_k drains while step k + 1 runs
                G, W = dev_buffers[2 + (k % 2)], dev_buffers[1]
            else:
                G, W = (dev_buffers[1], dev_buffers[2]) if k % 2 == 0 else (dev_buffers[2], dev_buffers[1])
            if k == 0:                                   # prologue: H2D(0) block-pipelined with the transform
                for c0, c1 in blocks:
                    h2d(0, c0, c1)
                    ev = torch.cuda.Event()
                    ev.record(hs)
                    s.wait_event(ev)
                    self._fwd_block(A[..., c0:c1], G, c0, c1, s)
            else:
                s.wait_event(h2d_done)
                if four and k >= 2:                      # G_k = G_{k-2} held Psi_{k-2}: drained a step ago
                    s.wait_event(d2h_events[k - 2])
                self._fwd_block(A, G, 0, nx, s)          # three buffers: G_k = W_{k-1}, dead since back(k-1)
            if k + 1 < n:                                # H2D(k+1) during factor_solve(k)
                fwd_done = torch.cuda.Event()
                fwd_done.record(s)
                hs.wait_event(fwd_done)
                for c0, c1 in [(0, nx)]:
                    h2d(k + 1, c0, c1)
                h2d_done = torch.cuda.Event()
                h2d_done.record(hs)
            if not four and d2h_done is not None:        # W_k = G_{k-1} holds Psi_{k-1} until drained
                s.wait_event(d2h_done)
            self._spatial_solves(G, W, nr, s)
            for c0, c1 in blocks:                        # back transform W -> G, D2H block-pipelined
                self._back_block(W, G[..., c0:c1], c0, c1, s)
                ev = torch.cuda.Event()
                ev.record(s)
                ds.wait_event(ev)
                N.check(lib.stfem_copy_cols(C.c_void_p(Ph[k].data_ptr() + 16 * c0), nx, N.ptr(G[..., c0:]), nx,
                                            c1 - c0, nr * nt, 1, N.stream_ptr(ds)))
            d2h_done = torch.cuda.Event()
            d2h_done.record(ds)
            d2h_events.append(d2h_done)
        s.wait_event(d2h_done)
        self.plan.check(s)        # one wait for the whole sequence
        return out_hosts


class BSSolver:
    """Bartels-Stewart variant: the fallback
    for a temporal core that is not diagonalizable.

    setup: complex Schur form C = X S X^H on the host (fp64, kappa2 = 1) +
    the same symbolic analysis as FD.  solve(F):
      (2) G = (Y (x) I) F                                   K3
      (3) for l = n_t-1 .. 0 (strictly sequential, SPEC.md Concurrency Model):
            (M_x + S[l,l] A_x) w_l = g_l                    K4/K5/K6, one shift
            g_l' -= S[l',l] A_x w_l  for every l' < l       bs_update_kernel
          (the incremental form of SPEC.md:418: A_x w_l formed once per l)
      (4) Psi = (X (x) I) W                                 K3
    All steps are stream-ordered GPU work; there is no CPU fallback."""

    def __init__(self, ops: SpatialOperators, M_t: np.ndarray, B_t: np.ndarray,
                 plan: SpatialPlan | None = None, leaf_size: int = 16):
        from .dense_complex_linalg import schur_factors
        t0 = time.perf_counter()
        self.ops = ops
        self.M_t = np.asarray(M_t, float)
        self.B_t = np.asarray(B_t, float)
        self.nt = self.M_t.shape[0]
        self.tf = schur_factors(self.M_t, self.B_t)
        t1 = time.perf_counter()
        self.plan = plan if plan is not None else SpatialPlan(ops, leaf_size)
        t2 = time.perf_counter()
        dev = ops.device
        self.X = torch.as_tensor(self.tf.X, dtype=C128, device=dev)
        self.Y = torch.as_tensor(self.tf.Y, dtype=C128, device=dev)
        self.diag = torch.as_tensor(np.diag(self.tf.S).copy(), dtype=C128, device=dev)
        # row l of S^T = column l of S: the coefficients scattered after step l
        self.St = torch.as_tensor(np.ascontiguousarray(self.tf.S.T), dtype=C128, device=dev)
        self.t_eig = t1 - t0
        self.t_symbolic = t2 - t1

    @property
    def kappa2(self) -> float:
        return self.tf.kappa2

    def solve(self, F: torch.Tensor, out: torch.Tensor | None = None, work: torch.Tensor | None = None,
              stream=None, timings: dict | None = None) -> torch.Tensor:
        N.require_cuda(F)
        nt, nx = self.nt, self.ops.n
        if F.shape[-2:] != (nt, nx):
            raise N.DimensionMismatch(N.ERR_DIM, f"solve: f {tuple(F.shape)} vs ({nt}, {nx})")
        if self.ops.Avals is None:
            raise RuntimeError("spatial operators are not assembled")
        single = F.dim() == 2
        Fb = (F.unsqueeze(0) if single else F).contiguous()
        nr = Fb.shape[0]
        G = _as_stack(out, Fb, "out") if out is not None else torch.empty_like(Fb)
        W = _as_stack(work, Fb, "work") if work is not None else torch.empty_like(Fb)
        if len({Fb.data_ptr(), G.data_ptr(), W.data_ptr()}) != 3:
            raise ValueError("solve: F, out and work must be three distinct buffers")
        s = stream if stream is not None else torch.cuda.current_stream()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if timings is not None else None
        if ev:
            ev[0].record(s)
        K.time_transform(self.Y, Fb, out=G, stream=s)                           # (2)
        if ev:
            ev[1].record(s)
        lay = blockvector_layout(nt, nx)
        lib = N.lib()
        self.plan.reserve(1, nr)          # no allocation (= no device sync) inside the sweep
        for l in range(nt - 1, -1, -1):                                          # (3)
            # stream-ordered sweep: n_t single-shift solves enqueued back to back, one error
            # check at the end that still names the sweep index l
            self.plan.set_shift_base(l)
            self.plan.factor_solve(self.diag[l:l + 1], G[:, l:l + 1], W[:, l:l + 1], lay, nr, stream=s,
                                   check=False)
            if l > 0:
                N.check(lib.stfem_bs_update(self.ops.handle, N.ptr(self.ops.Avals), N.ptr(W[:, l]),
                                            nt * nx, nr, N.ptr(self.St[l]), l, N.ptr(G), nt * nx, nx,
                                            N.stream_ptr(s)))
        self.plan.set_shift_base(0)
        if ev:
            ev[2].record(s)
        K.time_transform(self.X, W, out=G, stream=s)                            # (4)
        self.plan.check(s)
        if ev:
            ev[3].record(s)
            ev[3].synchronize()
            timings["forward_transform_s"] = ev[0].elapsed_time(ev[1]) / 1e3
            timings["sweep_s"] = ev[1].elapsed_time(ev[2]) / 1e3
            timings["back_transform_s"] = ev[2].elapsed_time(ev[3]) / 1e3
        if out is not None:
            return out
        return G[0] if single else G


def solve(ops: SpatialOperators, M_t: np.ndarray, B_t: np.ndarray, f: torch.Tensor,
          variant: SolverVariant = SolverVariant.FastDiagonalization, check_residual: bool = True,
          plan: SpatialPlan | None = None) -> SolveReport:
    """SPEC.md:374-382, both variants.  Times steps 1-4.  No
    silent fallback: FD on a defective core raises
    NotDiagonalizable and the caller retries with BartelsStewart."""
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if variant == SolverVariant.BartelsStewart:
        fdm = BSSolver(ops, M_t, B_t, plan=plan)
    else:
        fdm = FDMSolver(ops, M_t, B_t, plan=plan)
    timings = {"eig_s": fdm.t_eig, "symbolic_s": fdm.t_symbolic}
    psi = fdm.solve(f, timings=timings)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    res = relative_residual(ops, fdm.M_t, fdm.B_t, psi, f) if check_residual else None
    return SolveReport(psi, t1 - t0, fdm.kappa2, res, timings)
