"""Space-time error norms — host acceptance harness.

Untimed validation of a computed solution against a manufactured one: the
GPU solution is copied to the host once and integrated with the 7-point
degree-5 triangle rule x 5-point Gauss per space-time prism (SPEC.md:451,
:474).  P1 in space and time.  (GPU-resident error quadrature is §8(f) rank 1.)
"""

from __future__ import annotations

import math

import numpy as np

from .fem_assembly import gauss_legendre, triangle_rule
from .spatial_mesh import SpatialMesh
from .temporal_mesh import TemporalMesh

PI = math.pi


def eoc(errors):
    """log(e_{J-1}/e_J)/log 2."""
    e = np.asarray(errors, dtype=float)
    if e.size < 2 or (e <= 0).any():
        raise ValueError("eoc needs >= 2 positive errors")
    return list(np.log2(e[:-1] / e[1:]))


def exact_solution(name: str):
    """(psi, d_t psi, grad_x psi) callables for the configs' manufactured solutions."""
    s = lambda x, y: np.sin(PI * x) * np.sin(PI * y)              # noqa: E731
    sx = lambda x, y: PI * np.cos(PI * x) * np.sin(PI * y)        # noqa: E731
    sy = lambda x, y: PI * np.sin(PI * x) * np.cos(PI * y)        # noqa: E731
    if name == "sinpit":
        return (lambda x, y, t: s(x, y) * np.sin(PI * t) + 0j,
                lambda x, y, t: s(x, y) * PI * np.cos(PI * t) + 0j,
                lambda x, y, t: (sx(x, y) * np.sin(PI * t) + 0j, sy(x, y) * np.sin(PI * t) + 0j))
    if name == "texp":
        e = lambda t: np.exp(-1j * t)                              # noqa: E731
        return (lambda x, y, t: s(x, y) * t * e(t),
                lambda x, y, t: s(x, y) * e(t) * (1 - 1j * t),
                lambda x, y, t: (sx(x, y) * t * e(t), sy(x, y) * t * e(t)))
    if name == "paper":
        def psi(x, y, t):
            return np.exp(1j * t) * s(x, y) * np.sin(t * x * y)

        def dt(x, y, t):
            return np.exp(1j * t) * s(x, y) * (1j * np.sin(t * x * y) + x * y * np.cos(t * x * y))

        def grad(x, y, t):
            E, q, c = np.exp(1j * t), np.sin(t * x * y), np.cos(t * x * y)
            return (E * (sx(x, y) * q + s(x, y) * c * t * y), E * (sy(x, y) * q + s(x, y) * c * t * x))
        return psi, dt, grad
    raise KeyError(name)


def spacetime_errors_device(ops, mesh_t: TemporalMesh, coeffs, exact_name: str, psi0_nodal=None):
    """K8 on the GPU (§8(f) rank 1): same quadrature as `spacetime_errors`,
    for coefficients resident in HBM ((n_t, n_x) complex128 CUDA tensor)
    against one of the built-in manufactured solutions ('sinpit', 'texp',
    'paper').  psi0_nodal: (nv,) complex nodal values or None."""
    import ctypes as C

    import torch

    from . import _native as N
    from .fem_assembly import SOURCE_KINDS
    N.require_cuda(coeffs)
    if coeffs.dtype != torch.complex128 or coeffs.dim() != 2 or coeffs.stride(1) != 1:
        raise TypeError("coeffs must be a (n_t, n_x) complex128 tensor with unit column stride")
    bp = np.ascontiguousarray(mesh_t.breakpoints, dtype=np.float64)
    if coeffs.shape != (len(bp) - 1, ops.n):
        raise N.DimensionMismatch(N.ERR_DIM, f"coeffs {tuple(coeffs.shape)} vs ({len(bp) - 1}, {ops.n})")
    p0 = None
    if psi0_nodal is not None:
        p0 = torch.as_tensor(np.ascontiguousarray(psi0_nodal, dtype=np.complex128), device=coeffs.device)
    out = np.zeros(2)
    N.check(N.lib().stfem_spacetime_errors(ops.handle, SOURCE_KINDS[exact_name], bp.ctypes.data, len(bp) - 1,
                                           N.ptr(coeffs), coeffs.stride(0), N.ptr(p0), out.ctypes.data,
                                           N.stream_ptr()))
    return float(out[0]), float(out[1])


def spacetime_errors(coeffs: np.ndarray, exact, mesh_x: SpatialMesh, mesh_t: TemporalMesh,
                     psi0_nodal: np.ndarray | None = None):
    """(||psi - psi_h||_{L2(Q)}, |psi - psi_h|_{H1(Q)}) for P1 x P1 coefficients
    (n_t, n_x) (host array); psi_h = sum coeff phi_j phi_l (+ psi0)."""
    psi, dtpsi, grad = exact
    bp = mesh_t.breakpoints
    el = mesh_x.elements
    nv = mesh_x.num_vertices
    dof = mesh_x.interior_dof
    nodal = np.zeros((len(bp), nv), dtype=complex)
    inner = dof >= 0
    nodal[1:, inner] = np.asarray(coeffs)[:, dof[inner]]
    if psi0_nodal is not None:
        nodal += np.asarray(psi0_nodal)[None, :]
    qp, qw = triangle_rule()
    gt, gw = gauss_legendre(5)
    bary = np.column_stack([1 - qp[:, 0] - qp[:, 1], qp[:, 0], qp[:, 1]])     # (7,3)
    P = mesh_x.vertices[el]
    d1, d2 = P[:, 1] - P[:, 0], P[:, 2] - P[:, 0]
    area = 0.5 * (d1[:, 0] * d2[:, 1] - d1[:, 1] * d2[:, 0])
    gx = np.stack([P[:, 1, 1] - P[:, 2, 1], P[:, 2, 1] - P[:, 0, 1], P[:, 0, 1] - P[:, 1, 1]], 1) / (2 * area[:, None])
    gy = np.stack([P[:, 2, 0] - P[:, 1, 0], P[:, 0, 0] - P[:, 2, 0], P[:, 1, 0] - P[:, 0, 0]], 1) / (2 * area[:, None])
    Xq = np.tensordot(bary, P, axes=([1], [1])).transpose(1, 0, 2)          # (ne,7,2)
    xq, yq = Xq[..., 0], Xq[..., 1]
    wx = 2 * area[:, None] * qw[None, :]
    e2 = 0.0
    h2 = 0.0
    for k in range(len(bp) - 1):
        ht = bp[k + 1] - bp[k]
        U0, U1 = nodal[k][el], nodal[k + 1][el]
        dU = (U1 - U0) / ht
        for g in range(len(gt)):
            t = bp[k] + ht * gt[g]
            Ut = U0 + gt[g] * (U1 - U0)
            w = wx * (ht * gw[g])
            eu = psi(xq, yq, t) - Ut @ bary.T
            ed = dtpsi(xq, yq, t) - dU @ bary.T
            ex, ey = grad(xq, yq, t)
            ex = ex - np.sum(Ut * gx, 1)[:, None]
            ey = ey - np.sum(Ut * gy, 1)[:, None]
            e2 += float(np.sum(w * np.abs(eu) ** 2))
            h2 += float(np.sum(w * (np.abs(ed) ** 2 + np.abs(ex) ** 2 + np.abs(ey) ** 2)))
    return math.sqrt(e2), math.sqrt(h2)
