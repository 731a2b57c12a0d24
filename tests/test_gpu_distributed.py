"""GPU side of the multi-GPU FD path on one device: the factor kernels read
the all-to-all receive buffer (P, n_t/P, n_rhs, c) in place through the
chunked BlockVector layout (distributed.chunked_layout).  Emulates P ranks'
exchange with tensor reshapes and checks every shard's shifts against the
plain-layout solve (K4/K5/K6 through the C-ABI), bit for bit, with and
without spectral subtrees; plus a world-size-1 DistributedFDM solve."""
import numpy as np
import pytest
import torch

from paper_2504_07269_b200 import distributed as D
from paper_2504_07269_b200 import fem_assembly as fa
from paper_2504_07269_b200 import kronecker_solver as ks
from paper_2504_07269_b200 import spatial_mesh as sm
from paper_2504_07269_b200 import sparse_spatial_solver as sss
from paper_2504_07269_b200 import temporal_mesh as tm

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("spectral", [0, 64])
@pytest.mark.parametrize("P", [2, 4])
def test_chunked_receive_layout(P, spectral):
    ops = fa.assemble_spatial(sm.build_structured_square(24))   # n_x = 529: the last shard is zero padded
    nx = ops.n
    plan = sss.SpatialPlan(ops, spectral=spectral)
    nt, nr = 8, 3
    rng = np.random.default_rng(7)
    lam = rng.standard_normal(nt) * 0.1 - 1j * (0.05 + rng.random(nt))
    G = rng.standard_normal((nr, nt, nx)) + 1j * rng.standard_normal((nr, nt, nx))
    Gd = torch.from_numpy(G).cuda()
    W_ref = sss.factor_solve_batch(plan, lam, Gd).cpu().numpy()
    c = D.shard_cols(nx, P)
    ntl = nt // P
    for q in range(P):   # rank q's receive buffer: (P source ranks, ntl shifts, nr, c)
        R = torch.zeros((P, ntl, nr, c), dtype=torch.complex128, device="cuda")
        for src in range(P):
            lo, hi = src * c, min(nx, (src + 1) * c)
            R[src, :, :, :hi - lo] = Gd[:, q * ntl:(q + 1) * ntl, lo:hi].permute(1, 0, 2)
        Wq = torch.zeros_like(R)
        lam_q = torch.as_tensor(lam[q * ntl:(q + 1) * ntl], dtype=torch.complex128, device="cuda")
        plan.factor_solve(lam_q, R, Wq, D.chunked_layout(ntl, nr, c), nr)
        Wq = Wq.cpu().numpy()
        for src in range(P):
            lo, hi = src * c, min(nx, (src + 1) * c)
            got = Wq[src, :, :, :hi - lo].transpose(1, 0, 2)
            assert np.array_equal(got, W_ref[:, q * ntl:(q + 1) * ntl, lo:hi])


def test_distributed_world1_matches_fdm():
    mesh = sm.build_structured_square(24)
    ops = fa.assemble_spatial(mesh)
    tmesh = tm.uniform(1.0, 16)
    Mt, Bt = fa.assemble_temporal(tmesh)
    fdm = ks.FDMSolver(ops, Mt, Bt)
    rng = np.random.default_rng(1)
    F = torch.from_numpy(rng.standard_normal((2, 16, ops.n)) + 1j * rng.standard_normal((2, 16, ops.n))).cuda()
    ref = fdm.solve(F).cpu().numpy()
    solver = D.DistributedFDM(ops.n, 16, 2, fdm.X, fdm.Y, fdm.lam, D.CudaBackend(fdm.plan))
    out = D.unshard(solver.solve(D.shard_rhs(F, 0, 1)), ops.n, 0, 1).cpu().numpy()
    assert np.linalg.norm(out - ref) <= 1e-13 * np.linalg.norm(ref)


def test_fdm_solve_c_abi_matches_staged_path():
    """stfem_fdm_solve (one C call: the product path of FDMSolver.solve) = the three staged
    entry points (transform, factor_solve, transform), bit for bit; paired and plain K3."""
    mesh = sm.build_structured_square(24)
    ops = fa.assemble_spatial(mesh)
    Mt, Bt = fa.assemble_temporal(tm.uniform(1.0, 16))
    rng = np.random.default_rng(2)
    F = torch.from_numpy(rng.standard_normal((3, 16, ops.n)) + 1j * rng.standard_normal((3, 16, ops.n))).cuda()
    for paired in (True, False):
        fdm = ks.FDMSolver(ops, Mt, Bt, paired=paired)
        assert (fdm.pairs is not None) == paired
        one_call = fdm.solve(F)
        staged = fdm.solve(F, timings={})
        assert torch.equal(one_call, staged)


def test_native_comm_sharded_solve_world1():
    """stfem_comm_init (NCCL bound at run time, one rank) + the sharded branch of
    stfem_fdm_solve: shard layout (n_t, n_rhs, c), both exchanges through ncclSend/ncclRecv,
    factor + solve from the receive buffer's chunked layout."""
    mesh = sm.build_structured_square(24)
    ops = fa.assemble_spatial(mesh)
    Mt, Bt = fa.assemble_temporal(tm.uniform(1.0, 16))
    fdm = ks.FDMSolver(ops, Mt, Bt)
    rng = np.random.default_rng(3)
    F = torch.from_numpy(rng.standard_normal((2, 16, ops.n)) + 1j * rng.standard_normal((2, 16, ops.n))).cuda()
    ref = fdm.solve(F)
    comm = D.NativeComm()
    info = comm.info()
    assert info["nranks"] == 1 and info["rank"] == 0 and info["nccl_version"] >= 20000
    # the exchange itself: one rank sends its only block to itself
    a = torch.arange(10, dtype=torch.float64, device="cuda").to(torch.complex128)
    b = torch.zeros_like(a)
    comm.all_to_all(a, b)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    solver = D.NativeShardedFDM(fdm, 2, comm)
    out = D.unshard(solver.solve(D.shard_rhs(F, 0, 1)), ops.n, 0, 1).contiguous()
    assert torch.equal(out, ref)
    comm.close()
