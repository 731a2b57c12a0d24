"""Host setup of the spectral subtree elimination (spectral.py, K6) — CPU only.

For every subtree root the packed data must reproduce, for shifts spread over
the temporal spectrum, (a) the exact Schur complement the parent front
assembles, U(lam) = -K_GI K_II^{-1} K_IG, (b) the forward RHS contribution
r_Gam = -K_GI K_II^{-1} g_I and (c) the interior back-substitution
x_I = K_II^{-1} (g_I - K_IG x_Gam), exactly as csrc/spectral.cuh evaluates
them (U = -(R diag(w) R^T + C0 + lam C1), r = -(R (w o c) + Q c),
y = w o (c - R^T x) - Q^T x, x_I = V y, w = 1/(theta + lam), c = V^T g_I).
Also checks root selection (disjoint subtrees covering whole branches) and the
C-ABI round trip of stfem_plan_set_spectral (factor storage shrinks)."""
import numpy as np
import pytest

from oracle import stfem_oracle as O
from paper_2504_07269_b200 import fem_assembly as fa
from paper_2504_07269_b200 import spatial_mesh as sm
from paper_2504_07269_b200 import spectral as SP
from paper_2504_07269_b200.sparse_spatial_solver import SpatialPlan


def operators(mesh, deg):
    om = O.finish(2, mesh.vertices, mesh.elements)
    return O.assemble_spatial(om) if deg == 1 else O.assemble_spatial(om, 2, mesh.p2_elements)


CASES = {
    "square16": (lambda: sm.build_structured_square(16), 1, 40),
    "p2square6": (lambda: sm.refine_uniform(sm.build_structured_square(6)), 2, 60),
    "lshape6": (lambda: sm.build_lshape(6), 1, 50),
}


@pytest.mark.parametrize("name", list(CASES))
def test_spectral_formulas(name):
    make, deg, mcut = CASES[name]
    mesh = make()
    ops = fa.SpatialOperators(mesh, deg, device="cpu")
    plan = SpatialPlan(ops, spectral=0)
    Mx, Ax = operators(mesh, deg)
    fr, rows, perm = plan.fronts(), plan.front_rows(), plan.perm()
    data = SP.build(fr, rows, perm, Mx, Ax, mcut, threads=2)
    assert data.nroots >= 2
    Mp = Mx.toarray()[np.ix_(perm, perm)]
    Ap = Ax.toarray()[np.ix_(perm, perm)]
    # subtrees are disjoint and each interior is exactly the pivots of the root's subtree
    first = SP.subtree_first(fr)
    cover = np.zeros(ops.n, dtype=int)
    for t, f in enumerate(data.roots):
        assert data.first[t] == first[f]
        assert data.m[t] <= mcut and data.m[t] == fr[f, 0] + fr[f, 1] - first[f]
        par = fr[f, 3]
        assert par < 0 or fr[par, 0] + fr[par, 1] - first[par] > mcut
        cover[data.first[t]:data.first[t] + data.m[t]] += 1
    assert cover.max() == 1
    rng = np.random.default_rng(3)
    lams = [0.02 + 0.3j, 0.5 - 1e-9j, 3e-4 + 2e-3j, 0.1 + 0.0j]
    o = data.offsets.reshape(-1, 4)
    for t, f in enumerate(data.roots[:6]):
        m, g = int(data.m[t]), int(data.g[t])
        I = np.arange(data.first[t], data.first[t] + m)
        G = np.asarray(rows[f][fr[f, 1]:])
        V = data.V[o[t, 0]:o[t, 0] + m * m].reshape(m, m).T
        th = data.theta[o[t, 1]:o[t, 1] + m]
        R = data.RQ[o[t, 2]:o[t, 2] + g * m].reshape(m, g).T
        Q = data.RQ[o[t, 2] + g * m:o[t, 2] + 2 * g * m].reshape(m, g).T
        C0 = data.C01[o[t, 3]:o[t, 3] + g * g].reshape(g, g).T
        C1 = data.C01[o[t, 3] + g * g:o[t, 3] + 2 * g * g].reshape(g, g).T
        assert np.allclose(V.T @ Ap[np.ix_(I, I)] @ V, np.eye(m), atol=1e-10)
        for lam in lams:
            K_II = Mp[np.ix_(I, I)] + lam * Ap[np.ix_(I, I)]
            K_GI = Mp[np.ix_(G, I)] + lam * Ap[np.ix_(G, I)]
            w = 1.0 / (th + lam)
            U_ref = -K_GI @ np.linalg.solve(K_II, K_GI.T)
            U = -((R * w) @ R.T + C0 + lam * C1)
            assert np.linalg.norm(U - U_ref) <= 1e-12 * np.linalg.norm(U_ref) + 1e-300
            gI = rng.standard_normal(m) + 1j * rng.standard_normal(m)
            xG = rng.standard_normal(g) + 1j * rng.standard_normal(g)
            c = V.T @ gI
            r_ref = -K_GI @ np.linalg.solve(K_II, gI)
            r = -(R @ (w * c) + Q @ c)
            assert np.linalg.norm(r - r_ref) <= 1e-12 * np.linalg.norm(r_ref)
            x_ref = np.linalg.solve(K_II, gI - K_GI.T @ xG)
            y = w * (c - R.T @ xG) - Q.T @ xG
            assert np.linalg.norm(V @ y - x_ref) <= 1e-11 * np.linalg.norm(x_ref)


def test_set_spectral_abi():
    mesh = sm.build_structured_square(16)
    ops = fa.SpatialOperators(mesh, 1, device="cpu")
    plan = SpatialPlan(ops, spectral=0)
    Mx, Ax = operators(mesh, 1)
    base = plan.stats["factor_elems"]
    data = SP.build(plan.fronts(), plan.front_rows(), plan.perm(), Mx, Ax, 40, threads=1)
    SP.attach(plan.handle, data)
    st = SP.stats(plan.handle)
    assert st["nroots"] == data.nroots and st["bytes"] == data.nbytes()
    assert st["flops_u"] == sum(4 * (g * (g + 1) // 2) * m for m, g in zip(data.m, data.g))
    import ctypes as C
    from paper_2504_07269_b200 import _native as N
    s = N.plan_stats()
    N.check(N.lib().stfem_plan_stats_get(plan.handle, C.byref(s)))
    assert s.factor_elems < base
    # a mismatched interior range is rejected; nroots = 0 restores the plain plan
    bad = SP.SpectralData(data.roots, data.first + 1, data.offsets, data.V, data.theta, data.RQ, data.C01,
                          data.m, data.g)
    with pytest.raises(N.DimensionMismatch):
        SP.attach(plan.handle, bad)
    SP.attach(plan.handle, None)
    N.check(N.lib().stfem_plan_stats_get(plan.handle, C.byref(s)))
    assert s.factor_elems == base and SP.stats(plan.handle)["nroots"] == 0
