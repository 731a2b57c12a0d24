"""Generate golden mesh fixtures by importing the REFERENCE's own L0 modules
(`/root/reference/pkg/src/stfem/{spatial_mesh,temporal_mesh}.py`).

Run in the build container only (the reference does not exist on the GPU box):
    python tests/golden/make_golden.py
Writes tests/golden/meshes.npz.  The fixtures pin the oracle's and the
product's mesh numbering (spatial_mesh.py:51-70, :82-107, :121-156,
:205-215; temporal_mesh.py:49-77) to the reference bit for bit.
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from stfem import spatial_mesh as sm  # noqa: E402
from stfem import temporal_mesh as tm  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def lshape_text(n):
    """Vertex/element text for the L-shape convention, fed
    through the reference's mesh_from_text/_finish for boundary+numbering."""
    N = 2 * n
    xs = np.linspace(-1.0, 1.0, N + 1)
    keep = lambda i, j: not (i >= n and j < n)  # noqa: E731
    used = np.zeros((N + 1, N + 1), bool)
    for j in range(N):
        for i in range(N):
            if keep(i, j):
                used[j:j + 2, i:i + 2] = True
    vid = -np.ones((N + 1, N + 1), int)
    verts = []
    for j in range(N + 1):
        for i in range(N + 1):
            if used[j, i]:
                vid[j, i] = len(verts)
                verts.append((xs[i], xs[j]))
    tris = []
    for j in range(N):
        for i in range(N):
            if keep(i, j):
                a, b, c, d = vid[j, i], vid[j, i + 1], vid[j + 1, i], vid[j + 1, i + 1]
                tris += [(a, b, d), (a, d, c)]
    # boundary line is recomputed by _finish; write placeholder then patch
    tmp = sm._finish(2, np.array(verts), np.array(tris))
    return sm.mesh_to_text(tmp)


def dump(out, key, mesh):
    out[f"{key}/vertices"] = mesh.vertices
    out[f"{key}/elements"] = mesh.elements
    out[f"{key}/boundary"] = mesh.boundary
    out[f"{key}/interior_dof"] = mesh.interior_dof


def main():
    out = {}
    for m in (1, 2, 3, 4, 8, 16):
        dump(out, f"square{m}", sm.build_structured_square(m))
    for m in (1, 2, 4):
        r = sm.refine_uniform(sm.build_structured_square(m))
        dump(out, f"refine_square{m}", r)
    rr = sm.refine_uniform(sm.refine_uniform(sm.build_structured_square(2)))
    dump(out, "refine2_square2", rr)
    for m, L in ((2, 1.0), (4, 2.0), (5, 1.0)):
        dump(out, f"interval{m}_{L:g}", sm.build_interval(m, L))
    dump(out, "refine_interval4_2", sm.refine_uniform(sm.build_interval(4, 2.0)))
    for n in (1, 2, 4):
        dump(out, f"lshape{n}", sm.mesh_from_text(lshape_text(n)))
    out["mesh_size/square32"] = np.array(sm.mesh_size(sm.build_structured_square(32)))
    out["t/uniform5_64"] = tm.uniform(5.0, 64).breakpoints
    out["t/graded5_64_1.5"] = tm.graded(5.0, 64, 1.5).breakpoints
    out["t/bisect_graded5_64_1.5"] = tm.refine_bisect(tm.graded(5.0, 64, 1.5)).breakpoints
    out["t/uniform1_16"] = tm.uniform(1.0, 16).breakpoints
    out["t/uniform2_256"] = tm.uniform(2.0, 256).breakpoints
    np.savez_compressed(os.path.join(HERE, "meshes.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
