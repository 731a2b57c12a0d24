"""FEM assembly: spatial matrices and load vector on the GPU
(kernels K1/K2 of csrc/assembly.cu), temporal matrices on the host.

* `assemble_spatial(mesh, degree)` -> `SpatialOperators` holding the CSR
  pattern of M_x / A_x over interior DoFs and their values as device tensors
  (P1 closed forms, P2 = north-star extension).
* `assemble_temporal(tmesh, degree)` -> dense host (M_t, B_t) (SPEC.md:181-189,
  closed forms for P1; P2-in-time per SURVEY.md App. B).
* `assemble_rhs(ops, tmesh, source)` -> device (n_t, n_x) complex128 load vector
  (SPEC.md:190-198, 7-point x 5-point tensor quadrature, :217).
* `lifting_rhs(ops, tmesh, psi0_nodal)` -> -c_t (x) (A_x psi0).
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _native as N
from .spatial_mesh import SpatialMesh
from .temporal_mesh import TemporalMesh

SOURCE_KINDS = {"sinpit": 1, "texp": 2, "paper": 3}


class SparseRealMatrix:
    """CSR matrix whose values live on the GPU."""

    def __init__(self, rowptr: np.ndarray, colind: np.ndarray, values: torch.Tensor):
        self.rowptr = rowptr
        self.colind = colind
        self.values = values

    @property
    def shape(self):
        n = len(self.rowptr) - 1
        return (n, n)

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.values.detach().cpu().numpy(), self.colind, self.rowptr),
                             shape=self.shape)


class SpatialOperators:
    """Assembled spatial operators of one mesh (shared CSR pattern)."""

    def __init__(self, mesh: SpatialMesh, degree: int = 1, device="cuda"):
        if mesh.dimension != 2:
            raise ValueError("GPU assembly supports d = 2 meshes")
        if degree == 2 and mesh.p2_elements is None:
            raise ValueError("degree 2 needs a P2 node mesh (spatial_mesh.refine_uniform(parent))")
        self.mesh = mesh
        self.degree = degree
        self.n = mesh.num_dofs
        if self.n == 0:
            raise ValueError("assemble_spatial: mesh has no interior DoFs")
        els = mesh.elements if degree == 1 else mesh.p2_elements
        els = np.ascontiguousarray(els, dtype=np.int64)
        verts = np.ascontiguousarray(mesh.vertices, dtype=np.float64)
        dof = np.ascontiguousarray(mesh.interior_dof, dtype=np.int64)
        h = C.c_void_p()
        N.check(N.lib().stfem_asm_create(degree, len(verts), verts.ctypes.data, len(els),
                                         els.ctypes.data, dof.ctypes.data, C.byref(h)))
        self._h = h
        n32 = C.c_int32()
        nnz = C.c_int64()
        N.check(N.lib().stfem_asm_pattern(h, C.byref(n32), C.byref(nnz), None, None))
        self.rowptr = np.empty(self.n + 1, dtype=np.int64)
        self.colind = np.empty(nnz.value, dtype=np.int32)
        N.check(N.lib().stfem_asm_pattern(h, None, None, self.rowptr.ctypes.data, self.colind.ctypes.data))
        inner = np.flatnonzero(dof >= 0)
        self.coords = np.ascontiguousarray(verts[inner][np.argsort(dof[inner])])
        self.device = torch.device(device)
        self.Mvals = None
        self.Avals = None
        self.epoch = 0     # bumped by assemble(): consumers caching value-derived data compare it

    @property
    def handle(self):
        return self._h

    @property
    def nnz(self) -> int:
        return len(self.colind)

    def assemble(self, stream=None):
        """K1: fill M_x / A_x values on the GPU (coloured scatter)."""
        N.require_cuda()
        self.Mvals = torch.empty(self.nnz, dtype=torch.float64, device=self.device)
        self.Avals = torch.empty(self.nnz, dtype=torch.float64, device=self.device)
        N.check(N.lib().stfem_asm_spatial(self._h, N.ptr(self.Mvals), N.ptr(self.Avals),
                                          N.stream_ptr(stream)))
        self.epoch += 1
        return self

    @property
    def M_x(self) -> SparseRealMatrix:
        return SparseRealMatrix(self.rowptr, self.colind, self.Mvals)

    @property
    def A_x(self) -> SparseRealMatrix:
        return SparseRealMatrix(self.rowptr, self.colind, self.Avals)

    def spmv(self, which: str, v: torch.Tensor, alpha=1.0, out=None, stream=None) -> torch.Tensor:
        """alpha * (M_x or A_x) applied to each row of v ((k, n_x) complex128)."""
        vals = self.Mvals if which == "M" else self.Avals
        v2 = v.reshape(-1, self.n)
        if out is None:
            out = torch.empty_like(v2)
        a = complex(alpha)
        N.check(N.lib().stfem_csr_spmv_c(self._h, N.ptr(vals), N.ptr(v2), v2.stride(0), N.ptr(out),
                                         out.stride(0), v2.shape[0], a.real, a.imag, 0.0,
                                         N.stream_ptr(stream)))
        return out.reshape(v.shape)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and N is not None and N._lib is not None:
            N._lib.stfem_asm_destroy(h)
            self._h = None


def assemble_spatial(mesh: SpatialMesh, degree: int = 1, device="cuda") -> SpatialOperators:
    return SpatialOperators(mesh, degree, device).assemble()


def assemble_temporal(tmesh: TemporalMesh, degree: int = 1):
    """Dense host (M_t, B_t), row = test index."""
    h = tmesh.steps
    Nel = len(h)
    if degree == 1:
        M = np.zeros((Nel, Nel))
        B = np.zeros((Nel, Nel))
        idx = np.arange(Nel)
        M[idx, idx] = np.append((h[:-1] + h[1:]) / 3.0, h[-1] / 3.0)
        M[idx[:-1], idx[:-1] + 1] = h[1:] / 6.0
        M[idx[:-1] + 1, idx[:-1]] = h[1:] / 6.0
        B[idx[:-1], idx[:-1] + 1] = 0.5
        B[idx[:-1] + 1, idx[:-1]] = -0.5
        B[-1, -1] = 0.5
        return M, B
    if degree != 2:
        raise ValueError("temporal degree must be 1 or 2")
    n = 2 * Nel
    Mf = np.zeros((n + 1, n + 1))
    Bf = np.zeros((n + 1, n + 1))
    Ml = np.array([[4.0, 2.0, -1.0], [2.0, 16.0, 2.0], [-1.0, 2.0, 4.0]]) / 30.0
    Bl = np.array([[-0.5, 2 / 3, -1 / 6], [-2 / 3, 0.0, 2 / 3], [1 / 6, -2 / 3, 0.5]])
    for a in range(3):
        for b in range(3):
            rows = 2 * np.arange(Nel) + a
            cols = 2 * np.arange(Nel) + b
            np.add.at(Mf, (rows, cols), h * Ml[a, b])
            np.add.at(Bf, (rows, cols), Bl[a, b])
    return Mf[1:, 1:], Bf[1:, 1:]


def temporal_band(Mat: np.ndarray, bw: int) -> np.ndarray:
    """nt x (2bw+1) band storage band[l][k-l+bw] of a banded dense matrix."""
    nt = Mat.shape[0]
    out = np.zeros((nt, 2 * bw + 1))
    for o in range(-bw, bw + 1):
        l = np.arange(max(0, -o), min(nt, nt - o))
        out[l, o + bw] = Mat[l, l + o]
    return out


def temporal_load(tmesh: TemporalMesh) -> np.ndarray:
    """c_t[l] = int phi_l dt (P1): (h_l + h_{l+1})/2, last h_N/2."""
    h = tmesh.steps
    return np.append(0.5 * (h[:-1] + h[1:]), 0.5 * h[-1])


def assemble_rhs(ops: SpatialOperators, tmesh: TemporalMesh, source: str, out=None,
                 stream=None) -> torch.Tensor:
    """K2: F[l, j] = int int f phi_j phi_l for a built-in manufactured source."""
    if ops.degree != 1:
        raise ValueError("assemble_rhs: P1 space only (the P2 configs use Gaussian RHS)")
    kind = SOURCE_KINDS[source]
    nt = tmesh.num_elements
    if out is None:
        out = torch.empty((nt, ops.n), dtype=torch.complex128, device=ops.device)
    bp = np.ascontiguousarray(tmesh.breakpoints, dtype=np.float64)
    N.check(N.lib().stfem_asm_rhs(ops.handle, kind, bp.ctypes.data, nt, N.ptr(out), out.stride(0),
                                  N.stream_ptr(stream)))
    return out


def lifting_rhs(ops: SpatialOperators, tmesh: TemporalMesh, psi0: np.ndarray, out=None) -> torch.Tensor:
    """-(int phi_l dt) (A_x psi0)_j for psi0 given at interior DoFs (boundary
    zeroed).  The i<d_t psi0, .> term vanishes."""
    p = torch.as_tensor(np.ascontiguousarray(psi0, dtype=np.complex128), device=ops.device).reshape(1, -1)
    Ap = ops.spmv("A", p)
    c = torch.as_tensor(-temporal_load(tmesh), dtype=torch.float64, device=ops.device)
    res = c[:, None].to(torch.complex128) * Ap
    if out is not None:
        out.copy_(res)
        return out
    return res


def gauss_legendre(k: int = 5):
    """k-point Gauss rule on [0,1]."""
    if k < 1:
        raise ValueError("unsupported order")
    x, w = np.polynomial.legendre.leggauss(k)
    return 0.5 * (x + 1.0), 0.5 * w


def triangle_rule(degree: int = 5):
    """Degree-5, 7-point rule on the reference triangle, weights sum to 1/2."""
    if degree > 5:
        raise ValueError("unsupported degree")
    s = math.sqrt(15.0)
    a, b = (6 - s) / 21, (6 + s) / 21
    wa, wb = (155 - s) / 1200, (155 + s) / 1200
    pts = np.array([[1 / 3, 1 / 3], [a, a], [1 - 2 * a, a], [a, 1 - 2 * a],
                    [b, b], [1 - 2 * b, b], [b, 1 - 2 * b]])
    w = 0.5 * np.array([9 / 40, wa, wa, wa, wb, wb, wb])
    return pts, w
