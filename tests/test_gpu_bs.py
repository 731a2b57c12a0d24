"""GPU parity of the Bartels-Stewart variant
against the CPU oracle's restatement (oracle.bs_solve) on identical Schur
factors, against the FD variant, and of the sweep-update kernel
(stfem_bs_update) against numpy."""
import numpy as np
import pytest
import torch

from oracle import stfem_oracle as O
from paper_2504_07269_b200 import _native as N
from paper_2504_07269_b200 import fem_assembly as fa
from paper_2504_07269_b200 import kronecker_solver as ks
from paper_2504_07269_b200 import spatial_mesh as sm
from paper_2504_07269_b200 import temporal_mesh as tm

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def omesh(mesh):
    return O.finish(2, mesh.vertices, mesh.elements)


def test_bs_update_kernel_matches_numpy():
    mesh = sm.build_structured_square(9)
    ops = fa.assemble_spatial(mesh)
    nt, nx, nr, l = 1100, ops.n, 2, 1077          # l > 1024: two shared-memory chunks of S
    rng = np.random.default_rng(3)
    G = rng.standard_normal((nr, nt, nx)) + 1j * rng.standard_normal((nr, nt, nx))
    W = rng.standard_normal((nr, nt, nx)) + 1j * rng.standard_normal((nr, nt, nx))
    scol = rng.standard_normal(nt) + 1j * rng.standard_normal(nt)
    Gd, Wd, Sd = (torch.from_numpy(x).cuda() for x in (G, W, scol))
    N.check(N.lib().stfem_bs_update(ops.handle, N.ptr(ops.Avals), N.ptr(Wd[:, l]), nt * nx, nr, N.ptr(Sd), l,
                                    N.ptr(Gd), nt * nx, nx, N.stream_ptr()))
    A = ops.A_x.to_scipy()
    AW = (A @ W[:, l, :].T).T
    ref = G.copy()
    ref[:, :l, :] -= scol[:l][None, :, None] * AW[:, None, :]
    assert rel(Gd.cpu().numpy(), ref) < 1e-14


@pytest.mark.parametrize("kind,N,deg_t", [("square16", 16, 1), ("p2square6", 12, 1), ("lshape6", 10, 1),
                                          ("square12", 8, 2)])
def test_bs_solve_matches_oracle(kind, N, deg_t):
    """BS on the GPU vs the oracle's BS on identical Schur factors: <= 1e-9 per RHS,
    residual certificate <= 1e-8, and FD/BS agreement <= 1e-8 kappa_2."""
    if kind.startswith("p2"):
        mesh, deg = sm.refine_uniform(sm.build_structured_square(int(kind[8:]))), 2
        Mo, Ao = O.assemble_spatial(omesh(mesh), 2, mesh.p2_elements)
    elif kind.startswith("lshape"):
        mesh, deg = sm.build_lshape(int(kind[6:])), 1
        Mo, Ao = O.assemble_spatial(omesh(mesh))
    else:
        mesh, deg = sm.build_structured_square(int(kind[6:])), 1
        Mo, Ao = O.assemble_spatial(omesh(mesh))
    ops = fa.assemble_spatial(mesh, deg)
    Mt, Bt = fa.assemble_temporal(tm.uniform(1.0, N), deg_t)
    nt = Mt.shape[0]
    rng = np.random.default_rng(N)
    F = (rng.standard_normal((2, nt, ops.n)) + 1j * rng.standard_normal((2, nt, ops.n))) / np.sqrt(2)
    Fd = torch.from_numpy(F).cuda()
    bs = ks.BSSolver(ops, Mt, Bt)
    psi = bs.solve(Fd).cpu().numpy()
    sf = O.OSchurFactors(bs.tf.X, bs.tf.S, bs.tf.Y)       # identical host factors on both sides
    ref = O.bs_solve(Mo, Ao, sf, F)
    for r in range(2):
        assert rel(psi[r], ref[r]) < 1e-9, rel(psi[r], ref[r])
    assert ks.relative_residual(ops, Mt, Bt, torch.from_numpy(psi).cuda(), Fd) < 1e-8
    fd = ks.FDMSolver(ops, Mt, Bt)
    psi_fd = fd.solve(Fd).cpu().numpy()
    assert rel(psi_fd, psi) < 1e-8 * fd.kappa2


def test_bs_report_and_manufactured_errors():
    """solve(variant=BartelsStewart) on C1 reproduces the FD manufactured-solution
    errors (Table 1 and Table 2 report identical errors)."""
    from paper_2504_07269_b200 import error_analysis as ea
    mesh = sm.build_structured_square(16)
    tmesh = tm.uniform(1.0, 16)
    ops = fa.assemble_spatial(mesh)
    Mt, Bt = fa.assemble_temporal(tmesh)
    F = fa.assemble_rhs(ops, tmesh, "sinpit")
    rb = ks.solve(ops, Mt, Bt, F, variant=ks.SolverVariant.BartelsStewart)
    rf = ks.solve(ops, Mt, Bt, F)
    assert rb.kappa2 == 1.0 and rb.relative_residual < 1e-8
    eb = ea.spacetime_errors(rb.solution.cpu().numpy(), ea.exact_solution("sinpit"), mesh, tmesh)
    ef = ea.spacetime_errors(rf.solution.cpu().numpy(), ea.exact_solution("sinpit"), mesh, tmesh)
    for a, b in zip(eb, ef):
        assert abs(a - b) / b < 1e-6


def test_bs_c2_full_size():
    """C2 (64 x 64 P1, n_t = 64) at full size: BS vs FD, residual certificate."""
    from paper_2504_07269_b200.problems import Problem
    prob = Problem("C2", device="cuda")
    bs = ks.BSSolver(prob.ops, prob.M_t, prob.B_t)
    psi = bs.solve(prob.F)
    assert ks.relative_residual(prob.ops, prob.M_t, prob.B_t, psi, prob.F) < 1e-8
    fd = ks.FDMSolver(prob.ops, prob.M_t, prob.B_t)
    psi_fd = fd.solve(prob.F)
    assert rel(psi_fd.cpu().numpy(), psi.cpu().numpy()) < 1e-8 * fd.kappa2
