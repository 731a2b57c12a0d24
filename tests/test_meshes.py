"""Mesh numbering: product (vectorised) and oracle (loops) against golden
fixtures generated from the reference's own spatial_mesh / temporal_mesh
(tests/golden/make_golden.py)."""
import os

import numpy as np
import pytest

from oracle import stfem_oracle as O
from paper_2504_07269_b200 import spatial_mesh as sm
from paper_2504_07269_b200 import temporal_mesh as tm

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "meshes.npz"))


def same(mesh, key):
    assert np.array_equal(mesh.vertices, G[f"{key}/vertices"]), key
    assert np.array_equal(mesh.elements, G[f"{key}/elements"]), key
    assert np.array_equal(mesh.boundary, G[f"{key}/boundary"]), key
    assert np.array_equal(mesh.interior_dof, G[f"{key}/interior_dof"]), key


@pytest.mark.parametrize("m", [1, 2, 3, 4, 8, 16])
def test_square(m):
    same(sm.build_structured_square(m), f"square{m}")
    same(O.square_mesh(m), f"square{m}")


@pytest.mark.parametrize("m", [1, 2, 4])
def test_refine(m):
    r = sm.refine_uniform(sm.build_structured_square(m))
    same(r, f"refine_square{m}")
    ro, p2o = O.refine_mesh(O.square_mesh(m))
    same(ro, f"refine_square{m}")
    assert np.array_equal(r.p2_elements, p2o)
    # parent-with-midpoints table is consistent with the children of the reference
    ch = G[f"refine_square{m}/elements"].reshape(-1, 4, 3)
    p2g = np.stack([ch[:, 0, 0], ch[:, 1, 1], ch[:, 2, 2], ch[:, 0, 1], ch[:, 1, 2], ch[:, 0, 2]], 1)
    assert np.array_equal(r.p2_elements, p2g)


def test_refine_twice():
    same(sm.refine_uniform(sm.refine_uniform(sm.build_structured_square(2))), "refine2_square2")


@pytest.mark.parametrize("m,L", [(2, 1.0), (4, 2.0), (5, 1.0)])
def test_interval(m, L):
    same(sm.build_interval(m, L), f"interval{m}_{L:g}")
    same(O.interval_mesh(m, L), f"interval{m}_{L:g}")


def test_refine_interval():
    same(sm.refine_uniform(sm.build_interval(4, 2.0)), "refine_interval4_2")


@pytest.mark.parametrize("n", [1, 2, 4])
def test_lshape(n):
    same(sm.build_lshape(n), f"lshape{n}")
    same(O.lshape_mesh(n), f"lshape{n}")


def test_lshape_c5_count():
    assert sm.build_lshape(256).num_dofs == 195585


def test_c4_p2_count():
    assert sm.refine_uniform(sm.build_structured_square(256)).num_dofs == 261121


def test_mesh_size_and_text_roundtrip():
    assert sm.mesh_size(sm.build_structured_square(32)) == float(G["mesh_size/square32"])
    m = sm.build_lshape(2)
    m2 = sm.mesh_from_text(sm.mesh_to_text(m))
    assert np.array_equal(m2.vertices, m.vertices) and np.array_equal(m2.interior_dof, m.interior_dof)
    sm.check_admissible(m)
    sm.check_admissible(sm.refine_uniform(sm.build_structured_square(3)))


def test_temporal():
    assert np.array_equal(tm.uniform(5.0, 64).breakpoints, G["t/uniform5_64"])
    assert np.array_equal(tm.graded(5.0, 64, 1.5).breakpoints, G["t/graded5_64_1.5"])
    assert np.array_equal(tm.refine_bisect(tm.graded(5.0, 64, 1.5)).breakpoints,
                          G["t/bisect_graded5_64_1.5"])
    assert np.array_equal(tm.uniform(2.0, 256).breakpoints, G["t/uniform2_256"])
    assert np.array_equal(O.temporal_uniform(1.0, 16), G["t/uniform1_16"])
    with pytest.raises(ValueError):
        tm.TemporalMesh([0.0, 0.5, 0.5])
    with pytest.raises(ValueError):
        tm.graded(1.0, 4, 0.5)
    g = tm.graded(5.0, 64, 1.5)
    assert abs(g.max_step - 5 * (1 - (63 / 64) ** 1.5)) < 1e-12
