"""Host symbolic analysis (csrc/symbolic.cpp) — CPU only, through the C-ABI.

The fronts must cover the exact fill of L: for a dense no-pivot LDL^T of the
permuted matrix, every structurally nonzero L[i, j] must have row i in the
index list of the front that owns pivot j.  Also checks permutation validity,
postorder/parent consistency and nnz(L) bounds."""
import numpy as np
import pytest

from oracle import stfem_oracle as O
from paper_2504_07269_b200 import fem_assembly as fa
from paper_2504_07269_b200 import spatial_mesh as sm
from paper_2504_07269_b200.sparse_spatial_solver import SpatialPlan


def meshes():
    return {
        "square8": (sm.build_structured_square(8), 1),
        "square13": (sm.build_structured_square(13), 1),
        "p2square4": (sm.refine_uniform(sm.build_structured_square(4)), 2),
        "lshape4": (sm.build_lshape(4), 1),
        "lshape3": (sm.build_lshape(3), 1),
    }


@pytest.mark.parametrize("name", list(meshes()))
@pytest.mark.parametrize("leaf", [4, 32])
def test_fronts_cover_fill(name, leaf):
    mesh, deg = meshes()[name]
    ops = fa.SpatialOperators(mesh, deg, device="cpu")
    plan = SpatialPlan(ops, leaf_size=leaf)
    n = ops.n
    perm = plan.perm()
    assert np.array_equal(np.sort(perm), np.arange(n))
    fr = plan.fronts()
    rows = plan.front_rows()
    # pivots contiguous, postorder (children before parents), depth consistent
    assert fr[:, 1].sum() == n
    assert np.array_equal(np.cumsum(np.r_[0, fr[:-1, 1]]), fr[:, 0])
    for f, (pbeg, p, nf, parent, depth) in enumerate(fr):
        assert p >= 1 and nf == len(rows[f])
        assert np.array_equal(rows[f][:p], np.arange(pbeg, pbeg + p))
        assert np.all(np.diff(rows[f][p:]) > 0) and (p == nf or rows[f][p] >= pbeg + p)
        if parent >= 0:
            assert parent > f and fr[parent, 4] == depth - 1
            # child boundary rows belong to the parent front
            assert set(rows[f][p:]) <= set(rows[parent])
        else:
            assert depth == 0
    # exact fill of a no-pivot LDL^T of the permuted matrix
    if deg == 1:
        Mo, Ao = O.assemble_spatial(O.finish(2, mesh.vertices, mesh.elements))
    else:
        Mo, Ao = O.assemble_spatial(O.finish(2, mesh.vertices, mesh.elements), 2, mesh.p2_elements)
    K = (Mo + 0.37 * Ao).toarray()[np.ix_(perm, perm)]
    L = np.eye(n)
    A = K.copy()
    for j in range(n):
        d = A[j, j]
        L[j + 1:, j] = A[j + 1:, j] / d
        A[j + 1:, j + 1:] -= np.outer(L[j + 1:, j], A[j, j + 1:])
    owner = np.repeat(np.arange(len(fr)), fr[:, 1])
    nzi, nzj = np.nonzero(np.abs(np.tril(L, -1)) > 1e-13)
    for i, j in zip(nzi, nzj):
        assert i in set(rows[owner[j]]), (i, j)
    nnzL = int(np.count_nonzero(np.abs(np.tril(L)) > 1e-13))
    assert nnzL <= plan.stats["nnz_factor"]
    assert plan.stats["nnz_factor"] <= 2.0 * nnzL + n


def test_c3_c4_c5_plans_build():
    """Full-size symbolic analyses succeed and report sane statistics."""
    for m, deg in ((sm.build_structured_square(256), 1),
                   (sm.refine_uniform(sm.build_structured_square(256)), 2),
                   (sm.build_lshape(256), 1)):
        ops = fa.SpatialOperators(m, deg, device="cpu")
        plan = SpatialPlan(ops)
        st = plan.stats
        assert st["n"] == ops.n
        assert st["max_front"] <= 2200
        assert st["nnz_factor"] < 40 * ops.nnz
