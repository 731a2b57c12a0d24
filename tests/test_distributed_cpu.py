"""Multi-rank orchestration of the distributed FD solve on CPU (gloo, world 2
and 4): spatial sharding, (n_t, n_rhs, c) layouts, both all-to-alls and the
chunked BlockVector addressing the GPU factor kernel uses.  The compute
backend is a test stand-in built on the oracle (numpy transforms, SuperLU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import stfem_oracle as O
from paper_2504_07269_b200 import distributed as D


class OracleBackend:
    def __init__(self, Mx, Ax, nx):
        self.Mx, self.Ax, self.nx = Mx, Ax, nx

    def transform(self, T, x, out):
        out.copy_(T @ x)

    def factor_solve(self, lam, G, W, layout, nrhs):
        g = G.reshape(-1).numpy()
        w = W.reshape(-1).numpy()
        j = np.arange(self.nx)
        col = (j // layout.chunk_cols) * layout.chunk_stride + j % layout.chunk_cols
        for l in range(lam.numel()):
            for r in range(nrhs):
                idx = r * layout.rhs_stride + l * layout.shift_stride + col
                w[idx] = O._solve_shift(self.Mx, self.Ax, complex(lam[l]), g[idx])


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mesh = O.square_mesh(7)                       # n_x = 36 (not divisible by 4 -> padding)
        bp = O.temporal_uniform(1.0, 8)
        Mx, Ax = O.assemble_spatial(mesh)
        Mt, Bt = O.assemble_temporal(bp)
        tf = O.eigen_decompose(Mt, Bt)
        nx, nt, nr = Mx.shape[0], 8, 3
        rng = np.random.default_rng(0)
        F = rng.standard_normal((nr, nt, nx)) + 1j * rng.standard_normal((nr, nt, nx))
        X, Y, lam = D.broadcast_factors(tf.X if rank == 0 else np.zeros((nt, nt)),
                                        tf.Y if rank == 0 else np.zeros((nt, nt)),
                                        tf.lam if rank == 0 else np.zeros(nt), "cpu")
        solver = D.DistributedFDM(nx, nt, nr, X, Y, lam, OracleBackend(Mx, Ax, nx))
        Fp = D.shard_rhs(torch.from_numpy(F), rank, world)
        Psi_p = solver.solve(Fp)
        mine = D.unshard(Psi_p, nx, rank, world).numpy()
        ref = O.fdm_solve(Mx, Ax, tf, F)
        c = D.shard_cols(nx, world)
        lo, hi = rank * c, min(nx, (rank + 1) * c)
        err = np.linalg.norm(mine - ref[:, :, lo:hi]) / max(np.linalg.norm(ref[:, :, lo:hi]), 1e-300)
        q.put((rank, float(err)))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 4])
def test_distributed_fd_matches_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    res = [q.get(timeout=5) for _ in range(world)]
    assert all(p.exitcode == 0 for p in procs)
    for rank, err in res:
        assert err < 1e-12, (rank, err)


def test_layout_helpers():
    F = torch.arange(2 * 4 * 10, dtype=torch.float64).reshape(2, 4, 10).to(torch.complex128)
    parts = [D.unshard(D.shard_rhs(F, r, 3), 10, r, 3) for r in range(3)]
    assert torch.equal(torch.cat(parts, dim=2), F)
    lay = D.chunked_layout(2, 3, 5)
    assert (lay.rhs_stride, lay.shift_stride, lay.chunk_cols, lay.chunk_stride) == (5, 15, 5, 30)
