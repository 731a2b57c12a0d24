"""The five BASELINE.json configurations (plus the paper's level-0 preset).

Conventions:
  C1  square(16),  P1 x P1, T=1, N=16,   f from psi = s(x) sin(pi t)     + 1 Gaussian RHS
  C2  square(64),  P1 x P1, T=1, N=64,   same f                           + 1 Gaussian RHS
  C3  square(256), P1 x P1, T=2, N=256,  f from psi = s(x) t e^{-it}      + 1 Gaussian RHS
  C4  P2 nodes of square(256), P2 x P2, T=1, N=512 (1024 temporal DoFs), 1 Gaussian RHS
  C5  L-shape h=1/256, P1 x P1, T=1, N=1024, f=0, lifted wave packet psi0 + 8 Gaussian RHS
  paper0  square(32), T=5, N=64, the paper's manufactured solution
s(x) = sin(pi x1) sin(pi x2).  Gaussian RHS = (N(0,1) + i N(0,1))/sqrt(2),
drawn per block of 16 temporal rows x 8192 spatial columns from numpy
default_rng((seed, rhs, row block, column block)) (deterministic for any thread
count and any spatial sharding).  The public benchmark suite of the
paper is not used: these are the seeded synthetic stand-ins BASELINE.json
names.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np
import torch

from . import fem_assembly as fa
from . import spatial_mesh as sm
from . import temporal_mesh as tm

SEED = 20250409
ROWS_PER_CHUNK = 16


@dataclass(frozen=True)
class Config:
    name: str
    mesh: str            # "square:m" | "p2square:m" | "lshape:n"
    degree_x: int
    degree_t: int
    T: float
    N: int               # temporal elements
    source: str | None   # manufactured source name or None (f = 0)
    n_gauss: int
    psi0: str | None = None


CONFIGS = {
    "C1": Config("C1", "square:16", 1, 1, 1.0, 16, "sinpit", 1),
    "C2": Config("C2", "square:64", 1, 1, 1.0, 64, "sinpit", 1),
    "C3": Config("C3", "square:256", 1, 1, 2.0, 256, "texp", 1),
    "C4": Config("C4", "p2square:256", 2, 2, 1.0, 512, None, 1),
    "C5": Config("C5", "lshape:256", 1, 1, 1.0, 1024, None, 8, psi0="packet"),
    "paper0": Config("paper0", "square:32", 1, 1, 5.0, 64, "paper", 0),
}


def build_mesh(spec: str) -> sm.SpatialMesh:
    kind, arg = spec.split(":")
    m = int(arg)
    if kind == "square":
        return sm.build_structured_square(m)
    if kind == "p2square":
        return sm.refine_uniform(sm.build_structured_square(m))
    if kind == "lshape":
        return sm.build_lshape(m)
    raise KeyError(spec)


def wave_packet(x, y):
    """psi0 of configs[4]: exp(-|x - x0|^2 / (2 0.1^2) + 20 i x1), x0 = (-0.5, 0.5)."""
    return np.exp(-((x + 0.5) ** 2 + (y - 0.5) ** 2) / (2 * 0.1 ** 2) + 20j * x)


def psi0_interior(mesh: sm.SpatialMesh) -> np.ndarray:
    """Nodal psi0 at interior DoFs (boundary values zeroed)."""
    inner = np.flatnonzero(mesh.interior_dof >= 0)
    order = np.argsort(mesh.interior_dof[inner])
    v = mesh.vertices[inner[order]]
    return wave_packet(v[:, 0], v[:, 1])


COLS_PER_BLOCK = 8192


def gaussian_rhs(seed: int, n_rhs: int, nt: int, nx: int, out: np.ndarray | None = None,
                 threads: int | None = None, cols: tuple[int, int] | None = None) -> np.ndarray:
    """(n_rhs, nt, hi - lo) complex128 seeded Gaussian stack for the spatial columns
    cols = [lo, hi) (default: all n_x columns).  One RNG stream per (rhs, block of 16
    temporal rows, block of 8192 columns): every entry depends only on the seed and its
    own indices, so a spatial shard generates exactly its columns (no rank ever builds the
    full stack) and the result is the same for any thread count or sharding."""
    lo, hi = (0, nx) if cols is None else (max(0, cols[0]), min(nx, cols[1]))
    w = max(0, hi - lo)
    if out is None:
        out = np.empty((n_rhs, nt, w), dtype=np.complex128)
    assert out.shape == (n_rhs, nt, w)
    view = out.view(np.float64).reshape(n_rhs, nt, w, 2)
    jobs = [(r, c, b) for r in range(n_rhs) for c in range(0, nt, ROWS_PER_CHUNK)
            for b in range(lo // COLS_PER_BLOCK, -(-hi // COLS_PER_BLOCK) if w else 0)]
    scale = 1.0 / math.sqrt(2.0)

    def work(job):
        r, c0, b = job
        c1 = min(nt, c0 + ROWS_PER_CHUNK)
        b0, b1 = b * COLS_PER_BLOCK, min(nx, (b + 1) * COLS_PER_BLOCK)
        rng = np.random.default_rng((seed, r, c0 // ROWS_PER_CHUNK, b))
        re = rng.standard_normal((c1 - c0, b1 - b0))
        im = rng.standard_normal((c1 - c0, b1 - b0))
        s0, s1 = max(lo, b0), min(hi, b1)
        view[r, c0:c1, s0 - lo:s1 - lo, 0] = re[:, s0 - b0:s1 - b0] * scale
        view[r, c0:c1, s0 - lo:s1 - lo, 1] = im[:, s0 - b0:s1 - b0] * scale

    nthr = threads or min(32, len(os.sched_getaffinity(0)))
    if nthr > 1 and len(jobs) > 1:
        with ThreadPoolExecutor(nthr) as ex:
            list(ex.map(work, jobs))
    else:
        for j in jobs:
            work(j)
    return out


class Problem:
    """Meshes, assembled operators, temporal matrices and RHS stack for a config."""

    def __init__(self, cfg: Config | str, device="cuda", seed: int = SEED, with_rhs: bool = True,
                 rhs_host: bool = False):
        self.cfg = CONFIGS[cfg] if isinstance(cfg, str) else cfg
        c = self.cfg
        self.seed = seed
        self.mesh = build_mesh(c.mesh)
        self.tmesh = tm.uniform(c.T, c.N)
        self.ops = fa.SpatialOperators(self.mesh, c.degree_x, device)
        self.M_t, self.B_t = fa.assemble_temporal(self.tmesh, c.degree_t)
        self.nx = self.ops.n
        self.nt = self.M_t.shape[0]
        self.n_rhs = (1 if c.source else 0) + (1 if c.psi0 else 0) + c.n_gauss
        self.device = torch.device(device)
        self.F_host = None
        self.F = None
        self.psi0 = psi0_interior(self.mesh) if c.psi0 else None
        if with_rhs:
            self.build_rhs(host=rhs_host)

    @property
    def dofs(self) -> int:
        return self.nx * self.nt

    def assemble(self):
        self.ops.assemble()
        return self

    def build_rhs(self, host: bool = False):
        """F (n_rhs, n_t, n_x): [manufactured | lifted psi0] + Gaussian stack.
        The deterministic parts are assembled on the GPU (K2 / lifting); the
        Gaussian parts are generated on the host (pinned when host=True)."""
        c = self.cfg
        if self.ops.Mvals is None:
            self.assemble()
        det = []
        if c.source:
            det.append(fa.assemble_rhs(self.ops, self.tmesh, c.source))
        if c.psi0:
            det.append(fa.lifting_rhs(self.ops, self.tmesh, self.psi0))
        shape = (self.n_rhs, self.nt, self.nx)
        Fh = torch.empty(shape, dtype=torch.complex128, pin_memory=host and torch.cuda.is_available())
        if c.n_gauss:
            gaussian_rhs(self.seed, c.n_gauss, self.nt, self.nx, out=Fh.numpy()[len(det):])
        for i, d in enumerate(det):
            Fh[i].copy_(d.cpu())
        self.F_host = Fh
        self.F = Fh.to(self.device, non_blocking=False)
        return self.F

    def manufactured(self) -> str | None:
        return self.cfg.source
