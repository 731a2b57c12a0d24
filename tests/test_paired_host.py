"""Eigenpair pairing of the FD factors (paired_transform.py, the host half of
K3p) against dense numpy: pairing exists for every config's temporal pencil,
the numpy statements of the two kernels equal Y F and X W, and the FD solution
is invariant under the paired eigenbasis."""
import numpy as np
import pytest

from paper_2504_07269_b200 import dense_complex_linalg as dcl
from paper_2504_07269_b200 import fem_assembly as fa
from paper_2504_07269_b200 import paired_transform as PT
from paper_2504_07269_b200 import temporal_mesh as tm


def crand(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("N,deg,T", [(16, 1, 1.0), (64, 1, 1.0), (256, 1, 2.0), (512, 2, 1.0), (1024, 1, 1.0),
                                     (40, 2, 1.0)])
def test_config_pencils_pair(N, deg, T):
    Mt, Bt = fa.assemble_temporal(tm.uniform(T, N), deg)
    tf = dcl.temporal_factors(Mt, Bt)
    pf = PT.build(tf.eigenvalues, tf.X, Bt)
    assert pf is not None
    nt = Mt.shape[0]
    assert 2 * pf.npairs + pf.nself == nt
    # exact structure of the rebuilt basis
    for (l, p), s in zip(pf.rows_fwd, pf.scale_fwd):
        if p >= 0:
            assert pf.lam[p] == -np.conj(pf.lam[l])
            assert np.array_equal(pf.Y[p], s * np.conj(pf.Y[l]))
    # X' is still an eigenbasis of the core and Y' = X'^{-1} (i B)^{-1}
    Cc = dcl.form_temporal_core(Mt, Bt)
    assert rel(Cc @ pf.X, pf.X * pf.lam[None, :]) < 1e-12
    # (as accurate as LAPACK's own factors: ~kappa_2 eps, 1.0e-9 for tf at n_t = 1024)
    assert rel(pf.Y @ (1j * Bt) @ pf.X, np.eye(nt)) <= rel(tf.Y @ (1j * Bt) @ tf.X, np.eye(nt)) + 1e-13
    rng = np.random.default_rng(N)
    F = crand(rng, nt, 37)
    assert rel(PT.forward_host(pf, F), pf.Y @ F) < 1e-14
    assert rel(PT.back_host(pf, F), pf.X @ F) < 1e-14
    # FD invariance: X diag(1/(lam + mu)) Y f solves (M_t + mu i B_t) u = f with either basis
    mu = 3.7 + 0.2j
    exact = np.linalg.solve(Mt + mu * 1j * Bt, F)
    fd_old = tf.X @ ((tf.Y @ F) / (tf.eigenvalues + mu)[:, None])
    fd_new = PT.back_host(pf, PT.forward_host(pf, F) / (pf.lam + mu)[:, None])
    assert rel(fd_new, exact) <= 2 * rel(fd_old, exact) + 1e-14
    assert rel(fd_new, fd_old) < 1e-10


def synthetic(rng, npair, nself):
    """A real pencil-like structure: pairs (lam, -conj(lam)) with x_p = c conj(x_l) and
    self-paired purely imaginary eigenvalues with x = e^{i phi} r."""
    nt = 2 * npair + nself
    X = np.zeros((nt, nt), complex)
    lam = np.zeros(nt, complex)
    col = 0
    for _ in range(npair):
        x = crand(rng, nt)
        c = np.exp(1j * rng.uniform(0, 6.28))
        lam[col] = rng.uniform(0.5, 3) - 1j * rng.uniform(0.1, 2)
        lam[col + 1] = -np.conj(lam[col])
        X[:, col], X[:, col + 1] = x, c * np.conj(x)
        col += 2
    for _ in range(nself):
        lam[col] = -1j * rng.uniform(0.1, 2)
        X[:, col] = np.exp(1j * rng.uniform(0, 6.28)) * rng.standard_normal(nt)
        col += 1
    perm = rng.permutation(nt)
    B = rng.standard_normal((nt, nt)) + nt * np.eye(nt)
    return lam[perm], X[:, perm], B


@pytest.mark.parametrize("npair,nself", [(5, 0), (4, 2), (9, 6), (1, 0)])
def test_synthetic_pairs_and_self_pairs(npair, nself):
    rng = np.random.default_rng(10 * npair + nself)
    lam, X, B = synthetic(rng, npair, nself)
    pf = PT.build(lam, X, B)
    assert pf is not None and pf.npairs == npair and pf.nself == nself
    Y = np.linalg.solve(X, np.linalg.inv(1j * B))
    F = crand(rng, X.shape[0], 11)
    assert rel(PT.forward_host(pf, F), Y @ F) < 1e-12
    assert rel(PT.back_host(pf, F), X @ F) < 1e-12


def test_unpaired_spectrum_is_rejected():
    rng = np.random.default_rng(1)
    nt = 8
    lam = np.arange(1, nt + 1) * (1 - 0.5j)          # no lam_p = -conj(lam_l)
    X = crand(rng, nt, nt)
    assert PT.build(lam, X, np.eye(nt)) is None
    assert PT.build(lam[:7], X[:7, :7], np.eye(7)) is None   # odd n_t


def test_wrong_partner_vector_is_rejected():
    rng = np.random.default_rng(2)
    lam, X, B = synthetic(rng, 4, 0)
    X[:, 1] = crand(rng, 8)                          # breaks x_p = c conj(x_l) for one pair
    assert PT.build(lam, X, B) is None
