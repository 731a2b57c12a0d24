"""CPU-side checks of the product host code and the C-ABI library (no GPU)."""
import os
import re

import numpy as np
import pytest
import torch

from oracle import stfem_oracle as O
from paper_2504_07269_b200 import _native as N
from paper_2504_07269_b200 import dense_complex_linalg as dcl
from paper_2504_07269_b200 import fem_assembly as fa
from paper_2504_07269_b200 import problems
from paper_2504_07269_b200 import temporal_mesh as tm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "stfem_b200.h")).read()
    declared = set(re.findall(r"\b(stfem_[a-z0-9_]+)\s*\(", hdr))
    exported = set(N.exported_symbols())
    assert declared, "no declarations parsed"
    missing = declared - exported
    assert not missing, missing
    N.lib()  # loads without a GPU
    assert N.lib().stfem_version() == 1


def test_no_cpu_fallback_without_gpu():
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2504_07269_b200 import _kernels as K
    T = torch.eye(2, dtype=torch.complex128)
    with pytest.raises(N.NativeUnavailable):
        K.time_transform(T, torch.ones(2, 3, dtype=torch.complex128))


@pytest.mark.parametrize("deg", [1, 2])
def test_temporal_matrices_match_oracle(deg):
    for tmesh in (tm.uniform(2.0, 9), tm.graded(5.0, 12, 1.5)):
        M, B = fa.assemble_temporal(tmesh, deg)
        Mo, Bo = O.assemble_temporal(tmesh.breakpoints, deg)
        assert np.abs(M - Mo).max() < 1e-15 and np.abs(B - Bo).max() < 1e-15


def test_temporal_factors_match_oracle():
    for N_ in (16, 64, 256):
        Mt, Bt = fa.assemble_temporal(tm.uniform(1.0, N_))
        mine = dcl.temporal_factors(Mt, Bt)
        ref = O.eigen_decompose(Mt, Bt)
        assert np.abs(mine.eigenvalues - ref.lam).max() < 1e-15
        assert np.abs(mine.X - ref.X).max() < 1e-13
        assert abs(mine.kappa2 - ref.kappa2) / ref.kappa2 < 1e-12
        # SPEC.md:240 invariant: ||C - X S X^-1|| <= 1e-10 n_t ||C||
        C = dcl.form_temporal_core(Mt, Bt)
        R = C @ mine.X - mine.X @ mine.S
        assert np.linalg.norm(R) <= 1e-10 * N_ * np.linalg.norm(C) * mine.kappa2
        # Y = X^-1 (iB)^-1
        assert np.abs(mine.Y @ (1j * Bt) @ mine.X - np.eye(N_)).max() < 1e-9 * mine.kappa2


def test_not_diagonalizable_is_reported():
    with pytest.raises(dcl.NotDiagonalizable):
        dcl.eigen_decompose(np.array([[0.0, 1.0], [0.0, 0.0]]))


def test_eoc():
    from paper_2504_07269_b200.error_analysis import eoc
    assert np.allclose(eoc([4e-3, 1e-3]), [2.0])
    assert np.allclose(eoc([2.4e-1, 1.2e-1]), [1.0])
    with pytest.raises(ValueError):
        eoc([1.0, 0.0])


def test_gaussian_rhs_deterministic_across_threads():
    a = problems.gaussian_rhs(7, 2, 40, 33, threads=1)
    b = problems.gaussian_rhs(7, 2, 40, 33, threads=8)
    assert np.array_equal(a, b)
    assert abs(np.mean(np.abs(a) ** 2) - 1.0) < 0.1


def test_gaussian_rhs_column_shards_match_full_stack():
    """A spatial shard draws exactly its columns (multi-GPU ranks never build the full stack)."""
    full = problems.gaussian_rhs(3, 2, 40, 20000)
    for lo, hi in ((0, 2500), (5000, 17000), (17500, 20000), (8191, 8193)):
        part = problems.gaussian_rhs(3, 2, 40, 20000, cols=(lo, hi), threads=2)
        assert np.array_equal(full[:, :, lo:hi], part)


def test_config_sizes():
    """BASELINE.json configs: n_x and n_t."""
    want = {"C1": (225, 16), "C2": (3969, 64), "C3": (65025, 256), "C4": (261121, 1024), "C5": (195585, 1024)}
    for name, (nx, nt) in want.items():
        c = problems.CONFIGS[name]
        mesh = problems.build_mesh(c.mesh)
        assert mesh.num_dofs == nx
        assert c.degree_t * c.N == nt
