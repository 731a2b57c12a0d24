"""GPU uniform refinement: `refine_uniform` of
`spatial_mesh` on the device (csrc/mesh_refine.cu, C-ABI `stfem_mesh_refine2d`),
array-identical to the host builder and therefore to the reference
(/root/reference/pkg/src/stfem/spatial_mesh.py:121-156): same midpoint
numbering (first encounter of the edges), same children, same boundary flags
and interior-DoF numbering (tests/test_gpu_mesh.py).

The mesh type stays the host `SpatialMesh` (the assembly and the symbolic
analysis consume host arrays), so the refined arrays are copied back once.
1-D meshes have no shared edges to number and stay on the host builder.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from . import spatial_mesh as sm


def refine_uniform(mesh: sm.SpatialMesh, device: str = "cuda") -> sm.SpatialMesh:
    if mesh.dimension != 2:
        return sm.refine_uniform(mesh)
    N.require_cuda()
    nv, ne = mesh.num_vertices, mesh.num_elements
    dev = torch.device(device)
    verts = torch.as_tensor(np.ascontiguousarray(mesh.vertices, dtype=np.float64), device=dev)
    elems = torch.as_tensor(np.ascontiguousarray(mesh.elements, dtype=np.int64), device=dev)
    nvmax = nv + 3 * ne
    vout = torch.empty((nvmax, 2), dtype=torch.float64, device=dev)
    eout = torch.empty((4 * ne, 3), dtype=torch.int64, device=dev)
    p2 = torch.empty((ne, 6), dtype=torch.int64, device=dev)
    bnd = torch.empty(nvmax, dtype=torch.uint8, device=dev)
    dof = torch.empty(nvmax, dtype=torch.int64, device=dev)
    nvr, ndof = C.c_int32(), C.c_int32()
    with torch.cuda.device(dev):
        N.check(N.lib().stfem_mesh_refine2d(nv, N.ptr(verts), ne, N.ptr(elems), N.ptr(vout), N.ptr(eout), N.ptr(p2),
                                            N.ptr(bnd), N.ptr(dof), C.byref(nvr), C.byref(ndof),
                                            N.stream_ptr(None)))
    n = nvr.value
    return sm.SpatialMesh(2, vout[:n].cpu().numpy(), eout.cpu().numpy(), bnd[:n].cpu().numpy().astype(bool),
                          dof[:n].cpu().numpy(), p2.cpu().numpy())
