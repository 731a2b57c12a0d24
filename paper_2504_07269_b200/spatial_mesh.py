"""Spatial meshes with interior-DoF numbering (host side, numpy-vectorised).

Mirrors the reference module `stfem.spatial_mesh`
(/root/reference/pkg/src/stfem/spatial_mesh.py) — same type, same operation
names, same numbering contract — but every builder is vectorised so the
paper-scale meshes (m = 256 squares, P2 nodes of refine(square(256)), the
h = 1/256 L-shape) build in well under a second instead of seconds:

* `_finish`                 -> spatial_mesh.py:51-70 (boundary from edge counts,
                               interior DoFs numbered in vertex order)
* `build_structured_square` -> spatial_mesh.py:82-107
* `build_interval`          -> spatial_mesh.py:110-118
* `refine_uniform`          -> spatial_mesh.py:121-156 (midpoints appended in
                               first-encounter order; `p2_elements` exposes the
                               parent triangle + its 3 edge-midpoint nodes)
* `element_measures`, `mesh_size`, `check_admissible`, `mesh_to_text`,
  `mesh_from_text`          -> spatial_mesh.py:159-215

Array identity with the reference is asserted by tests/test_meshes.py against
golden fixtures generated from the reference itself.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class SpatialMesh:
    """Immutable conforming mesh (spatial_mesh.py:16-48)."""

    dimension: int
    vertices: np.ndarray
    elements: np.ndarray
    boundary: np.ndarray
    interior_dof: np.ndarray
    # P2 extension: (ne_parent, 6) node table (v0, v1, v2, m01, m12, m20) when
    # this mesh is the P2 node set of a parent triangulation.
    p2_elements: np.ndarray | None = field(default=None, compare=False)

    @property
    def num_vertices(self) -> int:
        return len(self.vertices)

    @property
    def num_elements(self) -> int:
        return len(self.elements)

    @property
    def num_dofs(self) -> int:
        return int((self.interior_dof >= 0).sum())


def _edge_keys(elements: np.ndarray, nv: int) -> np.ndarray:
    e = elements
    a = np.stack([e[:, 0], e[:, 1], e[:, 2]], 1).ravel()
    b = np.stack([e[:, 1], e[:, 2], e[:, 0]], 1).ravel()
    lo = np.minimum(a, b)
    hi = np.maximum(a, b)
    return lo * nv + hi


def _finish(dimension, vertices, elements, p2_elements=None) -> SpatialMesh:
    vertices = np.ascontiguousarray(vertices, dtype=float)
    elements = np.ascontiguousarray(elements, dtype=np.int64)
    nv = len(vertices)
    boundary = np.zeros(nv, dtype=bool)
    if dimension == 1:
        counts = np.bincount(elements.ravel(), minlength=nv)
        boundary[counts == 1] = True
    else:
        keys = _edge_keys(elements, nv)
        uk, cnt = np.unique(keys, return_counts=True)
        once = uk[cnt == 1]
        boundary[once // nv] = True
        boundary[once % nv] = True
    interior_dof = -np.ones(nv, dtype=np.int64)
    inner = np.flatnonzero(~boundary)
    interior_dof[inner] = np.arange(len(inner))
    if dimension == 1:
        vertices = vertices.reshape(-1, 1)
    return SpatialMesh(dimension, vertices, elements, boundary, interior_dof, p2_elements)


def build_structured_square(m: int) -> SpatialMesh:
    if m < 1:
        raise ValueError("m must be >= 1")
    xs = np.linspace(0.0, 1.0, m + 1)
    xg, yg = np.meshgrid(xs, xs, indexing="xy")
    vertices = np.column_stack([xg.ravel(), yg.ravel()])
    j, i = np.meshgrid(np.arange(m), np.arange(m), indexing="ij")
    v00 = (j * (m + 1) + i).ravel()
    v10, v01, v11 = v00 + 1, v00 + m + 1, v00 + m + 2
    tris = np.empty((2 * m * m, 3), dtype=np.int64)
    tris[0::2] = np.stack([v00, v10, v11], 1)
    tris[1::2] = np.stack([v00, v11, v01], 1)
    return _finish(2, vertices, tris)


def build_interval(m: int, length: float) -> SpatialMesh:
    if m < 1:
        raise ValueError("m must be >= 1")
    if length <= 0:
        raise ValueError("length must be positive")
    vertices = np.linspace(0.0, length, m + 1)
    elements = np.column_stack([np.arange(m), np.arange(1, m + 1)])
    return _finish(1, vertices, elements)


def build_lshape(n: int) -> SpatialMesh:
    """L-shaped (-1,1)^2 minus [0,1)x(-1,0] with h = 1/n: a 2n x 2n cell grid,
    the removed quadrant's cells dropped, grid vertices used by kept cells
    numbered lexicographically by (row, column), each cell split like
    `build_structured_square` (BASELINE configs[4])."""
    N = 2 * n
    xs = np.linspace(-1.0, 1.0, N + 1)
    jj, ii = np.meshgrid(np.arange(N + 1), np.arange(N + 1), indexing="ij")
    used = ~((ii > n) & (jj < n))
    vid = -np.ones((N + 1, N + 1), dtype=np.int64)
    vid[used] = np.arange(int(used.sum()))
    vertices = np.column_stack([xs[ii[used]], xs[jj[used]]])
    cj, ci = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    keep = ~((ci >= n) & (cj < n))
    cj, ci = cj[keep], ci[keep]
    v00, v10 = vid[cj, ci], vid[cj, ci + 1]
    v01, v11 = vid[cj + 1, ci], vid[cj + 1, ci + 1]
    tris = np.empty((2 * len(cj), 3), dtype=np.int64)
    tris[0::2] = np.stack([v00, v10, v11], 1)
    tris[1::2] = np.stack([v00, v11, v01], 1)
    return _finish(2, vertices, tris)


def refine_uniform(mesh: SpatialMesh) -> SpatialMesh:
    nv = mesh.num_vertices
    if mesh.dimension == 1:
        el = mesh.elements
        ne = len(el)
        mid = nv + np.arange(ne)
        x = mesh.vertices[:, 0]
        verts = np.concatenate([x, 0.5 * (x[el[:, 0]] + x[el[:, 1]])])
        elems = np.empty((2 * ne, 2), dtype=np.int64)
        elems[0::2] = np.stack([el[:, 0], mid], 1)
        elems[1::2] = np.stack([mid, el[:, 1]], 1)
        return _finish(1, verts, elems)
    el = mesh.elements
    ne = len(el)
    keys = _edge_keys(el, nv)                      # encounter order: e0:(01,12,20), e1:...
    uk, first, inv = np.unique(keys, return_index=True, return_inverse=True)
    rank = np.empty(len(uk), dtype=np.int64)
    rank[np.argsort(first, kind="stable")] = np.arange(len(uk))
    mid_id = (nv + rank[inv]).reshape(ne, 3)       # m01, m12, m20
    order = np.argsort(first, kind="stable")
    lo, hi = uk[order] // nv, uk[order] % nv
    P = mesh.vertices
    newv = np.column_stack([(P[lo, 0] + P[hi, 0]) / 2, (P[lo, 1] + P[hi, 1]) / 2])
    verts = np.concatenate([P, newv])
    v0, v1, v2 = el[:, 0], el[:, 1], el[:, 2]
    m01, m12, m20 = mid_id[:, 0], mid_id[:, 1], mid_id[:, 2]
    elems = np.empty((4 * ne, 3), dtype=np.int64)
    elems[0::4] = np.stack([v0, m01, m20], 1)
    elems[1::4] = np.stack([m01, v1, m12], 1)
    elems[2::4] = np.stack([m20, m12, v2], 1)
    elems[3::4] = np.stack([m01, m12, m20], 1)
    p2 = np.stack([v0, v1, v2, m01, m12, m20], 1)
    return _finish(2, verts, elems, p2)


def p2_mesh(parent: SpatialMesh) -> SpatialMesh:
    """P2 node mesh of a parent triangulation: the vertices of
    refine_uniform(parent), interior numbering from its _finish, and
    `p2_elements` = parent triangles with their edge-midpoint nodes."""
    return refine_uniform(parent)


def element_measures(mesh: SpatialMesh) -> np.ndarray:
    pts = mesh.vertices[mesh.elements]
    if mesh.dimension == 1:
        return pts[:, 1, 0] - pts[:, 0, 0]
    e1 = pts[:, 1] - pts[:, 0]
    e2 = pts[:, 2] - pts[:, 0]
    return 0.5 * (e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0])


def mesh_size(mesh: SpatialMesh) -> float:
    meas = element_measures(mesh)
    if mesh.dimension == 1:
        return float(meas.max())
    return float(np.sqrt(meas.max()))


def check_admissible(mesh: SpatialMesh) -> None:
    meas = element_measures(mesh)
    assert (meas > 0).all(), "non-positive element measure"
    if mesh.dimension == 2:
        _, cnt = np.unique(_edge_keys(mesh.elements, mesh.num_vertices), return_counts=True)
        assert ((cnt == 1) | (cnt == 2)).all(), "edge shared by more than two elements"
    rebuilt = _finish(mesh.dimension, mesh.vertices, mesh.elements)
    assert (rebuilt.boundary == mesh.boundary).all(), "stale boundary flags"
    dofs = np.sort(mesh.interior_dof[mesh.interior_dof >= 0])
    assert (dofs == np.arange(mesh.num_dofs)).all(), "dof numbering gap"


def mesh_to_text(mesh: SpatialMesh) -> str:
    """Plain-text exchange format (SPEC.md spatial_mesh External Interfaces):
    "d nv ne", vertex rows, 0-based element rows, one boundary-flag row."""
    out = [f"{mesh.dimension} {mesh.num_vertices} {mesh.num_elements}"]
    out.extend(map(lambda v: " ".join(map(repr, map(float, v))), mesh.vertices))
    out.extend(map(lambda e: " ".join(map(str, map(int, e))), mesh.elements))
    out.append(" ".join(np.where(mesh.boundary, "1", "0")))
    return "\n".join(out) + "\n"


def mesh_from_text(text: str) -> SpatialMesh:
    """Inverse of mesh_to_text; boundary flags must match the connectivity."""
    lines = [ln for ln in text.strip().splitlines() if ln.strip()]
    d, nv, ne = map(int, lines[0].split())
    coords = np.array([ln.split() for ln in lines[1:1 + nv]], dtype=float)
    conn = np.array([ln.split() for ln in lines[1 + nv:1 + nv + ne]], dtype=np.int64)
    mesh = _finish(d, coords if d == 2 else coords[:, 0], conn)
    stored = np.array(lines[1 + nv + ne].split()) == "1"
    if stored.shape != mesh.boundary.shape or np.any(stored != mesh.boundary):
        raise ValueError("boundary flags in file disagree with connectivity")
    return mesh
