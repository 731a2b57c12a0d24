"""GPU uniform refinement (csrc/mesh_refine.cu) against the host builder, which the golden
fixtures pin to the reference (tests/test_meshes.py): every array identical."""
import time

import numpy as np
import pytest

from paper_2504_07269_b200 import spatial_mesh as sm
from paper_2504_07269_b200 import spatial_mesh_gpu as smg

pytestmark = pytest.mark.gpu


def same(a: sm.SpatialMesh, b: sm.SpatialMesh):
    assert a.dimension == b.dimension
    for f in ("vertices", "elements", "boundary", "interior_dof", "p2_elements"):
        x, y = getattr(a, f), getattr(b, f)
        if x is None or y is None:
            assert x is None and y is None, f
            continue
        assert x.shape == y.shape and x.dtype == y.dtype, f
        assert np.array_equal(x, y), f


@pytest.mark.parametrize("name", ["square1", "square7", "square64", "lshape12", "square5x2"])
def test_refine_matches_host(name):
    if name.startswith("lshape"):
        mesh = sm.build_lshape(int(name[6:]))
    elif name.endswith("x2"):
        mesh = sm.refine_uniform(sm.build_structured_square(int(name[6:-2])))   # refine a refined mesh
    else:
        mesh = sm.build_structured_square(int(name[6:]))
    got = smg.refine_uniform(mesh)
    same(got, sm.refine_uniform(mesh))
    sm.check_admissible(got)


def test_refine_c4_size_and_time():
    """The C4 mesh (P2 nodes of square(256)): identical arrays; the device part is timed."""
    mesh = sm.build_structured_square(256)
    smg.refine_uniform(mesh)   # warm-up (library load, allocator)
    t0 = time.perf_counter()
    got = smg.refine_uniform(mesh)
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    ref = sm.refine_uniform(mesh)
    t_host = time.perf_counter() - t0
    same(got, ref)
    assert got.num_dofs == 261121
    print(f"refine_uniform(square(256)): gpu {t_gpu * 1e3:.1f} ms (with copies), host {t_host * 1e3:.1f} ms")


def test_interval_falls_back_to_host():
    mesh = sm.build_interval(9, 2.0)
    same(smg.refine_uniform(mesh), sm.refine_uniform(mesh))
