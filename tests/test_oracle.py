"""Pin the CPU oracle (oracle/stfem_oracle.py) to the reference's known answers:
SPEC.md examples and the paper's published Table 2 / Table 3 numbers
(PAPER.md:214-218, :237), plus the survey-time values of SURVEY.md App. A."""
import math

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import stfem_oracle as O


def test_spec_spatial_examples():
    M, A = O.assemble_spatial(O.square_mesh(2))
    assert np.allclose(M.toarray(), [[1 / 8]], atol=1e-16) and np.allclose(A.toarray(), [[4]], atol=1e-15)
    M, A = O.assemble_spatial(O.interval_mesh(2, 1.0))
    assert np.allclose(M.toarray(), [[1 / 3]]) and np.allclose(A.toarray(), [[4]])
    M, A = O.assemble_spatial(O.square_mesh(6))
    x = np.random.default_rng(0).standard_normal(M.shape[0])
    assert x @ (A @ x) > 0 and x @ (M @ x) > 0
    assert abs(M - M.T).max() < 1e-17 and abs(A - A.T).max() < 1e-15


def test_spec_temporal_examples():
    h = 0.7
    M, B = O.assemble_temporal(np.array([0.0, h]))
    assert np.allclose(M, [[h / 3]]) and np.allclose(B, [[0.5]])
    M, B = O.assemble_temporal(np.array([0.0, h, 2 * h]))
    assert np.allclose(M, [[2 * h / 3, h / 6], [h / 6, h / 3]]) and np.allclose(B, [[0, 0.5], [-0.5, 0.5]])
    for deg in (1, 2):                                        # SPEC.md:189 (+ P2)
        bp = np.sort(np.r_[0.0, np.random.default_rng(deg).random(9).cumsum()])
        M, B = O.assemble_temporal(bp, deg)
        E = np.zeros_like(B)
        E[-1, -1] = 1.0
        assert np.abs(B + B.T - E).max() < 1e-15


def test_temporal_closed_forms_vs_quadrature():
    """SPEC.md:545 property: closed forms vs a degree-5 quadrature oracle <= 1e-13."""
    bp = np.r_[0.0, np.cumsum(np.random.default_rng(3).random(6) + 0.1)]
    for deg in (1, 2):
        M, B = O.assemble_temporal(bp, deg)
        x, w = O.gauss_rule(5)
        n = M.shape[0]
        Mq = np.zeros((n, n))
        Bq = np.zeros((n, n))
        tdofs = O.temporal_dof_times(bp, deg)
        nodes = np.r_[0.0, tdofs]
        for e in range(len(bp) - 1):
            t = bp[e] + (bp[e + 1] - bp[e]) * x
            ww = (bp[e + 1] - bp[e]) * w
            # Lagrange basis on all nodes restricted to element e
            loc = [k for k in range(len(nodes)) if bp[e] - 1e-14 <= nodes[k] <= bp[e + 1] + 1e-14]
            for a in loc:
                pa = np.ones_like(t)
                da = np.zeros_like(t)
                others = [nodes[c] for c in loc if c != a]
                for i, o in enumerate(others):
                    pa = pa * (t - o) / (nodes[a] - o)
                for i, o in enumerate(others):
                    term = np.ones_like(t) / (nodes[a] - o)
                    for j, o2 in enumerate(others):
                        if j != i:
                            term = term * (t - o2) / (nodes[a] - o2)
                    da = da + term
                for b in loc:
                    pb = np.ones_like(t)
                    for o in [nodes[c] for c in loc if c != b]:
                        pb = pb * (t - o) / (nodes[b] - o)
                    if a > 0 and b > 0:
                        Mq[b - 1, a - 1] += np.sum(ww * pa * pb)
                        Bq[b - 1, a - 1] += np.sum(ww * da * pb)
        assert np.abs(M - Mq).max() < 1e-13 and np.abs(B - Bq).max() < 1e-13


def test_quadrature_rules():
    x, w = O.gauss_rule(5)
    assert abs(np.sum(w * x ** 9) - 0.1) < 1e-14
    p, w = O.triangle_rule()
    assert abs(w.sum() - 0.5) < 1e-15
    for a in range(6):
        for b in range(6 - a):
            exact = math.factorial(a) * math.factorial(b) / math.factorial(a + b + 2)
            assert abs(np.sum(w * p[:, 0] ** a * p[:, 1] ** b) - exact) < 1e-15


def test_spec_dense_linalg_examples():
    h = 0.4
    M, B = O.assemble_temporal(np.array([0.0, h]))
    C = O.form_temporal_core(M, B)
    assert np.allclose(C, [[-2j * h / 3]])
    tf = O.eigen_decompose(M, B)
    assert np.allclose(tf.lam, [-2j * h / 3]) and np.allclose(tf.X, [[1]]) and tf.kappa2 == 1.0  # :270
    X = np.array([[1.0, 1.0], [0.0, 1.0]])
    s = np.linalg.svd(X, compute_uv=False)
    assert abs(s[0] / s[1] - (3 + math.sqrt(5)) / 2) < 1e-12


def test_spec_global_1x1():
    """psi = 1/(4/3 + i/16)."""
    Mx, Ax = O.assemble_spatial(O.square_mesh(2))
    Mt, Bt = O.assemble_temporal(np.array([0.0, 1.0]))
    tf = O.eigen_decompose(Mt, Bt)
    psi = O.fdm_solve(Mx, Ax, tf, np.array([[1.0 + 0j]]))
    assert abs(psi[0, 0] - 1 / (4 / 3 + 1j / 16)) < 1e-15
    assert abs(O.apply_global(Mx, Ax, Mt, Bt, np.array([[1.0 + 0j]]))[0, 0] - (4 / 3 + 1j / 16)) < 1e-15


@pytest.mark.parametrize("m,N,graded", [(2, 3, False), (3, 5, True), (4, 4, False), (3, 8, True)])
def test_fd_vs_dense_oracle(m, N, graded):
    """SPEC.md:539 acceptance 1: FD vs explicit Kronecker system <= 1e-10."""
    mesh = O.square_mesh(m)
    bp = O.temporal_graded(1.0, N, 1.5) if graded else O.temporal_uniform(1.0, N)
    Mx, Ax = O.assemble_spatial(mesh)
    Mt, Bt = O.assemble_temporal(bp)
    f = np.random.default_rng(m * N).standard_normal((N, Mx.shape[0])) * (1 + 1j)
    psi = O.fdm_solve(Mx, Ax, O.eigen_decompose(Mt, Bt), f)
    ref = np.linalg.solve(O.dense_global(Mx, Ax, Mt, Bt), f.ravel()).reshape(f.shape)
    assert np.linalg.norm(psi - ref) / np.linalg.norm(ref) < 1e-10


def test_kappa2_table2():
    """PAPER.md:214-216 kappa_2(X_t) column, T=5, within 5%, T-independence."""
    for N, k in ((64, 2.3e2), (128, 7.0e2), (256, 2.2e3)):
        Mt, Bt = O.assemble_temporal(O.temporal_uniform(5.0, N))
        kap = O.eigen_decompose(Mt, Bt).kappa2
        assert abs(kap - k) / k < 0.05
        assert f"{kap:.1e}" == f"{k:.1e}"
    ks = [O.eigen_decompose(*O.assemble_temporal(O.temporal_uniform(T, 64))).kappa2 for T in (1, 5, 10)]
    assert max(ks) / min(ks) - 1 < 1e-6


def test_eigen_pairing_and_sign():
    """Im(lambda) <= 0 and pairs (lam, -conj(lam))."""
    Mt, Bt = O.assemble_temporal(O.temporal_uniform(1.0, 64))
    lam = O.eigen_decompose(Mt, Bt).lam
    assert (lam.imag <= 1e-14).all()
    for l in lam:
        assert np.min(np.abs(lam + np.conj(l))) < 1e-12


def _paper_level(m, N, bp=None):
    mesh = O.square_mesh(m)
    bp = O.temporal_uniform(5.0, N) if bp is None else bp
    Mx, Ax = O.assemble_spatial(mesh)
    Mt, Bt = O.assemble_temporal(bp)
    psi, dt, gr, f = O.manufactured("paper")
    F = O.assemble_rhs(mesh, bp, f)
    tf = O.eigen_decompose(Mt, Bt)
    coeffs = O.fdm_solve(Mx, Ax, tf, F, threads=O.cpu_threads())
    res = np.linalg.norm(O.apply_global(Mx, Ax, Mt, Bt, coeffs) - F) / np.linalg.norm(F)
    return O.spacetime_errors(mesh, bp, coeffs, psi, dt, gr), tf.kappa2, res


def test_paper_table2_row1():
    """n = 61504, L2 3.2e-03, H1 2.4e-01, kappa 2.3e+02 (printed digits)."""
    (l2, h1), kap, res = _paper_level(32, 64)
    assert f"{l2:.1e}" == "3.2e-03" and f"{h1:.1e}" == "2.4e-01" and f"{kap:.1e}" == "2.3e+02"
    assert abs(l2 - 3.1900e-03) < 5e-8 and abs(h1 - 2.3969e-01) < 5e-6
    assert res < 1e-8


@pytest.mark.slow
def test_paper_table2_row2():
    """n = 508032, L2 8.1e-04, H1 1.2e-01, kappa 7.0e+02; eoc ~2 / ~1."""
    (l2, h1), kap, _ = _paper_level(64, 128)
    assert f"{l2:.1e}" == "8.1e-04" and f"{h1:.1e}" == "1.2e-01" and f"{kap:.1e}" == "7.0e+02"
    e = O.eoc([3.1900e-03, l2])
    assert 1.8 <= e[0] <= 2.2


def test_paper_table3_row1_graded():
    """graded q=1.5, L2 3.2e-03, kappa 1.1e+02, h_t 1.2e-01."""
    bp = O.temporal_graded(5.0, 64, 1.5)
    assert f"{np.diff(bp).max():.1e}" == "1.2e-01"
    (l2, h1), kap, _ = _paper_level(32, 64, bp)
    assert f"{l2:.1e}" == "3.2e-03" and f"{kap:.1e}" == "1.1e+02"


def test_survey_c1_errors():
    """C1 manufactured errors 4.004296e-03 / 1.670489e-01."""
    mesh = O.square_mesh(16)
    bp = O.temporal_uniform(1.0, 16)
    Mx, Ax = O.assemble_spatial(mesh)
    Mt, Bt = O.assemble_temporal(bp)
    psi, dt, gr, f = O.manufactured("sinpit")
    F = O.assemble_rhs(mesh, bp, f)
    c = O.fdm_solve(Mx, Ax, O.eigen_decompose(Mt, Bt), F)
    l2, h1 = O.spacetime_errors(mesh, bp, c, psi, dt, gr)
    assert f"{l2:.6e}" == "4.004296e-03" and f"{h1:.6e}" == "1.670489e-01"


def test_manufactured_sources_consistent():
    """SPEC.md:434 ExactSolution invariant: f = i d_t psi - lap psi (finite differences)."""
    rng = np.random.default_rng(0)
    pts = rng.random((50, 3))
    for name in ("sinpit", "texp", "paper"):
        psi, dt, gr, f = O.manufactured(name)
        hh = 1e-4
        for x, y, t in pts:
            lap = (psi(x + hh, y, t) + psi(x - hh, y, t) + psi(x, y + hh, t) + psi(x, y - hh, t)
                   - 4 * psi(x, y, t)) / hh ** 2
            dtn = (psi(x, y, t + hh) - psi(x, y, t - hh)) / (2 * hh)
            assert abs(dtn - dt(x, y, t)) < 1e-6
            assert abs(1j * dt(x, y, t) - lap - f(x, y, t)) < 1e-5


def test_p2_spatial_sanity():
    """P2 operators on the full node set: 1'M1 = |Omega|, A 1 = 0."""
    mesh, p2 = O.refine_mesh(O.square_mesh(4))
    full = O.OMesh(2, mesh.vertices, mesh.elements, np.zeros(len(mesh.vertices), bool),
                   np.arange(len(mesh.vertices)))
    M, A = O.assemble_spatial(full, 2, p2)
    one = np.ones(M.shape[0])
    assert abs(one @ (M @ one) - 1.0) < 1e-14
    assert np.abs(A @ one).max() < 1e-13
    x2 = mesh.vertices[:, 0] ** 2
    assert isinstance(M, sp.csr_matrix)
    inner = ~O.finish(2, mesh.vertices, mesh.elements).boundary
    assert np.abs((A @ x2 + 2 * (M @ one))[inner]).max() < 1e-12


# ---------------------------------------------------------------------------
# Bartels-Stewart variant
# ---------------------------------------------------------------------------

def test_bs_spec_global_1x1():
    """both variants give psi = 1/(4/3 + i/16) on the 1 x 1 system."""
    Mx, Ax = O.assemble_spatial(O.square_mesh(2))
    Mt, Bt = O.assemble_temporal(np.array([0.0, 1.0]))
    psi = O.bs_solve(Mx, Ax, O.schur_decompose(Mt, Bt), np.array([[1.0 + 0j]]))
    assert abs(psi[0, 0] - 1 / (4 / 3 + 1j / 16)) < 1e-15


@pytest.mark.parametrize("m,N,graded", [(2, 3, False), (3, 5, True), (4, 4, False), (3, 8, True)])
def test_bs_vs_dense_oracle(m, N, graded):
    """the BS variant matches the explicit Kronecker system <= 1e-10."""
    mesh = O.square_mesh(m)
    bp = O.temporal_graded(1.0, N, 1.5) if graded else O.temporal_uniform(1.0, N)
    Mx, Ax = O.assemble_spatial(mesh)
    Mt, Bt = O.assemble_temporal(bp)
    f = np.random.default_rng(m * N + 1).standard_normal((2, N, Mx.shape[0])) * (1 - 2j)
    psi = O.bs_solve(Mx, Ax, O.schur_decompose(Mt, Bt), f)
    D = O.dense_global(Mx, Ax, Mt, Bt)
    for r in range(2):
        ref = np.linalg.solve(D, f[r].ravel()).reshape(f[r].shape)
        assert np.linalg.norm(psi[r] - ref) / np.linalg.norm(ref) < 1e-10


def test_bs_fd_variant_agreement():
    """BS and FD agree within 1e-8 kappa_2(X_t) (C1 sizes, P1 in time)."""
    mesh = O.square_mesh(16)
    Mx, Ax = O.assemble_spatial(mesh)
    Mt, Bt = O.assemble_temporal(O.temporal_uniform(1.0, 16))
    f = np.random.default_rng(7).standard_normal((16, Mx.shape[0])) + 0.5j
    tf = O.eigen_decompose(Mt, Bt)
    a = O.fdm_solve(Mx, Ax, tf, f)
    b = O.bs_solve(Mx, Ax, O.schur_decompose(Mt, Bt), f)
    assert np.linalg.norm(a - b) / np.linalg.norm(b) < 1e-8 * tf.kappa2


@pytest.mark.parametrize("N,deg", [(16, 1), (64, 1), (32, 2)])
def test_host_schur_decompose(N, deg):
    """unitarity, residual, triangularity, kappa2 = 1, and the
    Schur diagonal equals the eigenvalues of the core within 1e-8."""
    from paper_2504_07269_b200 import dense_complex_linalg as dl
    from paper_2504_07269_b200 import fem_assembly as fa
    from paper_2504_07269_b200 import temporal_mesh as tm
    Mt, Bt = fa.assemble_temporal(tm.uniform(1.0, N), deg)
    n = Mt.shape[0]
    C = dl.form_temporal_core(Mt, Bt)
    sf = dl.schur_factors(Mt, Bt)
    X, S = sf.X, sf.S
    assert np.linalg.norm(X.conj().T @ X - np.eye(n)) <= 1e-12 * n
    assert np.linalg.norm(C - X @ S @ X.conj().T) <= 1e-10 * n * np.linalg.norm(C)
    assert np.abs(np.tril(S, -1)).max() == 0.0 and sf.kappa2 == 1.0 and sf.variant == "schur"
    assert np.allclose(sf.Y @ (1j * Bt), X.conj().T, atol=1e-12)
    ev = np.sort_complex(dl.temporal_factors(Mt, Bt).eigenvalues)
    assert np.abs(np.sort_complex(np.diag(S)) - ev).max() < 1e-8
    oracle = O.schur_decompose(Mt, Bt)
    assert np.abs(np.sort_complex(np.diag(oracle.S)) - ev).max() < 1e-8


@pytest.mark.parametrize("kind", ["square7", "p2square5", "lshape4"])
def test_vectorised_assembly_equals_loop_assembly(kind):
    """The full-size parity tests use assemble_spatial_vec; pin it to the loop restatement."""
    from paper_2504_07269_b200 import spatial_mesh as sm
    if kind.startswith("p2"):
        mesh = sm.refine_uniform(sm.build_structured_square(int(kind[8:])))
        om = O.finish(2, mesh.vertices, mesh.elements)
        Ml, Al = O.assemble_spatial(om, 2, mesh.p2_elements)
        Mv, Av = O.assemble_spatial_vec(mesh.vertices, mesh.p2_elements, mesh.interior_dof, 2)
    else:
        mesh = sm.build_lshape(int(kind[6:])) if kind.startswith("lshape") else sm.build_structured_square(int(kind[6:]))
        om = O.finish(2, mesh.vertices, mesh.elements)
        Ml, Al = O.assemble_spatial(om)
        Mv, Av = O.assemble_spatial_vec(mesh.vertices, mesh.elements, mesh.interior_dof, 1)
    for a, b in ((Ml, Mv), (Al, Av)):
        a.sort_indices()
        assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
        assert np.abs(a.data - b.data).max() <= 4e-16 * np.abs(a.data).max() * 8


def test_nd_superlu_mode_equals_default_mode():
    """The timing baseline's second SuperLU mode (shared ND ordering, no pivoting) solves the same system."""
    from paper_2504_07269_b200 import spatial_mesh as sm
    mesh = sm.build_structured_square(12)
    om = O.finish(2, mesh.vertices, mesh.elements)
    M, A = O.assemble_spatial(om)
    rng = np.random.default_rng(0)
    perm = rng.permutation(M.shape[0])
    b = rng.standard_normal(M.shape[0]) + 1j * rng.standard_normal(M.shape[0])
    for lam in (0.3 - 0.1j, -0.01 - 1e-5j):
        x0 = O._solve_shift(M, A, lam, b)
        x1 = O._solve_shift_nd(M, A, lam, b, perm)
        assert np.linalg.norm(x0 - x1) <= 1e-11 * np.linalg.norm(x0)
