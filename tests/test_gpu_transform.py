"""K3 time-axis transform (DMMA complex GEMM) vs numpy."""
import numpy as np
import pytest
import torch

from paper_2504_07269_b200 import _kernels as K

pytestmark = pytest.mark.gpu


def crand(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


@pytest.mark.parametrize("nt,ncols", [(1, 1), (3, 2), (16, 450), (17, 65), (64, 7938),
                                      (100, 333), (256, 4096)])
def test_transform_matches_numpy(nt, ncols):
    rng = np.random.default_rng(nt * 1000 + ncols)
    T = crand(rng, nt, nt)
    v = crand(rng, nt, ncols)
    ref = T @ v
    out = K.time_transform(torch.from_numpy(T).cuda(), torch.from_numpy(v).cuda()).cpu().numpy()
    err = np.linalg.norm(out - ref) / np.linalg.norm(ref)
    assert err < 1e-14, err


def test_transform_batched_strided():
    rng = np.random.default_rng(7)
    nt, n = 48, 300
    T = crand(rng, nt, nt)
    v = crand(rng, 3, nt, n)
    vt = torch.from_numpy(v).cuda()
    out = K.time_transform(torch.from_numpy(T).cuda(), vt).cpu().numpy()
    ref = np.einsum("lk,bkj->blj", T, v)
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) < 1e-14
    # strided rows (a column slice of a wider array)
    wide = crand(rng, nt, 2 * n)
    sl = torch.from_numpy(wide).cuda()[:, 5:5 + n]
    out2 = K.time_transform(torch.from_numpy(T).cuda(), sl).cpu().numpy()
    ref2 = T @ wide[:, 5:5 + n]
    assert np.linalg.norm(out2 - ref2) / np.linalg.norm(ref2) < 1e-14


def test_transform_identity_and_diag():
    """SPEC.md:398-399 examples: T = I leaves v unchanged; diag scales blocks."""
    rng = np.random.default_rng(3)
    v = crand(rng, 2, 5)
    I = np.eye(2, dtype=complex)
    out = K.time_transform(torch.from_numpy(I).cuda(), torch.from_numpy(v).cuda()).cpu().numpy()
    assert np.array_equal(out, v)
    D = np.diag([2.0, 3.0]).astype(complex)
    out = K.time_transform(torch.from_numpy(D).cuda(), torch.from_numpy(v).cuda()).cpu().numpy()
    assert np.allclose(out, np.diag([2.0, 3.0]) @ v, rtol=0, atol=1e-15)


# ---- K3p: eigenpair-paired transforms (paired_transform.py) ----
from paper_2504_07269_b200 import dense_complex_linalg as dcl  # noqa: E402
from paper_2504_07269_b200 import fem_assembly as fa  # noqa: E402
from paper_2504_07269_b200 import paired_transform as PT  # noqa: E402
from paper_2504_07269_b200 import temporal_mesh as tm  # noqa: E402


def _pairs(N, deg, T=1.0):
    Mt, Bt = fa.assemble_temporal(tm.uniform(T, N), deg)
    tf = dcl.temporal_factors(Mt, Bt)
    pf = PT.build(tf.eigenvalues, tf.X, Bt)
    assert pf is not None
    return pf, PT.DevicePairs(pf, "cuda")


@pytest.mark.parametrize("N,deg,ncols", [(16, 1, 450), (64, 1, 7938), (256, 1, 4097), (512, 2, 3000),
                                         (1024, 1, 700), (40, 2, 65), (8, 1, 1)])
def test_paired_transforms_match_dense(N, deg, ncols):
    pf, dp = _pairs(N, deg)
    nt = pf.X.shape[0]
    rng = np.random.default_rng(N + ncols)
    F = crand(rng, nt, ncols)
    G = K.transform_pair_fwd(dp, torch.from_numpy(F).cuda()).cpu().numpy()
    ref = pf.Y @ F
    assert np.linalg.norm(G - ref) / np.linalg.norm(ref) < 1e-14
    W = torch.from_numpy(F).cuda()
    P = K.transform_pair_back(dp, W).cpu().numpy()
    ref = pf.X @ F
    assert np.linalg.norm(P - ref) / np.linalg.norm(ref) < 1e-14


def test_paired_transforms_batched_strided():
    pf, dp = _pairs(48, 1)
    nt, n = pf.X.shape[0], 300
    rng = np.random.default_rng(5)
    v = crand(rng, 3, nt, n)
    G = K.transform_pair_fwd(dp, torch.from_numpy(v).cuda()).cpu().numpy()
    ref = np.einsum("lk,bkj->blj", pf.Y, v)
    assert np.linalg.norm(G - ref) / np.linalg.norm(ref) < 1e-14
    wide = crand(rng, 2, nt, 2 * n)
    full = torch.from_numpy(wide).cuda()
    sl = full[..., 7:7 + n]
    out = torch.empty((2, nt, n), dtype=torch.complex128, device="cuda")
    K.transform_pair_back(dp, sl, out=out)
    ref = np.einsum("lk,bkj->blj", pf.X, wide[..., 7:7 + n])
    got = out.cpu().numpy()
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-14
    # columns outside the slice are untouched by the in-place pre-pass
    back = full.cpu().numpy()
    assert np.array_equal(back[..., :7], wide[..., :7]) and np.array_equal(back[..., 7 + n:], wide[..., 7 + n:])


def test_paired_transform_self_pairs():
    """Purely imaginary (self-paired) eigenvalues: x = e^{i phi} r, one output row per source."""
    rng = np.random.default_rng(11)
    npair, nself = 13, 6
    nt = 2 * npair + nself
    X = np.zeros((nt, nt), complex)
    lam = np.zeros(nt, complex)
    for q in range(npair):
        x = crand(rng, nt)
        lam[2 * q] = rng.uniform(0.5, 3) - 1j * rng.uniform(0.1, 2)
        lam[2 * q + 1] = -np.conj(lam[2 * q])
        X[:, 2 * q], X[:, 2 * q + 1] = x, np.exp(0.3j * q) * np.conj(x)
    for q in range(nself):
        lam[2 * npair + q] = -1j * (q + 1)
        X[:, 2 * npair + q] = np.exp(0.7j * q) * rng.standard_normal(nt)
    B = rng.standard_normal((nt, nt)) + nt * np.eye(nt)
    pf = PT.build(lam, X, B)
    assert pf is not None and pf.nself == nself
    dp = PT.DevicePairs(pf, "cuda")
    F = crand(rng, nt, 333)
    G = K.transform_pair_fwd(dp, torch.from_numpy(F).cuda()).cpu().numpy()
    Y = np.linalg.solve(X, np.linalg.inv(1j * B))
    assert np.linalg.norm(G - Y @ F) / np.linalg.norm(Y @ F) < 1e-13
    P = K.transform_pair_back(dp, torch.from_numpy(F).cuda()).cpu().numpy()
    assert np.linalg.norm(P - X @ F) / np.linalg.norm(X @ F) < 1e-13


@pytest.mark.parametrize("N,deg,ncols", [(64, 1, 450), (256, 1, 4097), (40, 2, 65)])
def test_paired_transforms_column_maps(N, deg, ncols):
    """stfem_transform_pair_fwd_map scatters its result columns (out_cols), stfem_pair_mix +
    stfem_transform_pair_back_map gathers its operand columns (in_cols): with a permutation and
    its use as both maps the pair reproduces the unmapped transforms column for column
    (bit-identical: the same arithmetic per column), also on column blocks of a wider stack."""
    pf, dp = _pairs(N, deg)
    nt = pf.X.shape[0]
    rng = np.random.default_rng(N + ncols)
    F = torch.from_numpy(crand(rng, nt, ncols)).cuda()
    iperm = torch.from_numpy(rng.permutation(ncols).astype(np.int32)).cuda()
    G_ref = K.transform_pair_fwd(dp, F)
    G = torch.full_like(F, float("nan"))
    c_mid = ncols // 3
    for c0, c1 in ((0, c_mid), (c_mid, ncols)):          # column blocks of F into the whole of G
        K.transform_pair_fwd(dp, F[:, c0:c1], out=G, out_cols=iperm[c0:c1])
    assert torch.equal(G[:, iperm.long()], G_ref)
    P_ref = K.transform_pair_back(dp, G_ref.clone())
    K.pair_mix(dp, G)
    P = torch.empty_like(F)
    for c0, c1 in ((0, c_mid), (c_mid, ncols)):
        K.transform_pair_back(dp, G, out=P[:, c0:c1], in_cols=iperm[c0:c1], mixed=True)
    assert torch.equal(P, P_ref)
    with pytest.raises(Exception):
        K.transform_pair_back(dp, G, out=P, in_cols=iperm)            # a map needs the pre-pass first
