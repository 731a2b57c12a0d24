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
