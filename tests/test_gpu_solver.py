"""GPU parity: assembly (K1/K2), multifrontal factor+solve (K4/K5), FD solve,
apply_global (K7) against the CPU oracle on the same inputs."""
import numpy as np
import pytest
import torch

from oracle import stfem_oracle as O
from paper_2504_07269_b200 import fem_assembly as fa
from paper_2504_07269_b200 import kronecker_solver as ks
from paper_2504_07269_b200 import spatial_mesh as sm
from paper_2504_07269_b200 import sparse_spatial_solver as sss
from paper_2504_07269_b200 import temporal_mesh as tm
from paper_2504_07269_b200.dense_complex_linalg import temporal_factors

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def omesh(mesh):
    return O.finish(2, mesh.vertices, mesh.elements)


@pytest.mark.parametrize("kind", ["square7", "p2square5", "lshape3"])
def test_assembly_matches_oracle(kind):
    if kind == "square7":
        mesh, deg = sm.build_structured_square(7), 1
        Mo, Ao = O.assemble_spatial(omesh(mesh))
    elif kind == "p2square5":
        mesh, deg = sm.refine_uniform(sm.build_structured_square(5)), 2
        Mo, Ao = O.assemble_spatial(omesh(mesh), 2, mesh.p2_elements)
    else:
        mesh, deg = sm.build_lshape(3), 1
        Mo, Ao = O.assemble_spatial(omesh(mesh))
    ops = fa.assemble_spatial(mesh, deg)
    M = ops.M_x.to_scipy().toarray()
    A = ops.A_x.to_scipy().toarray()
    assert rel(M, Mo.toarray()) < 1e-14
    assert rel(A, Ao.toarray()) < 1e-14


def test_spec_example_m2():
    """m=2 -> M_x = [1/8], A_x = [4]."""
    ops = fa.assemble_spatial(sm.build_structured_square(2))
    assert abs(ops.Mvals.item() - 1 / 8) < 1e-15 and abs(ops.Avals.item() - 4) < 1e-14


@pytest.mark.parametrize("source", ["sinpit", "texp", "paper"])
def test_rhs_matches_oracle(source):
    mesh = sm.build_structured_square(6)
    bp = O.temporal_uniform(1.5, 5)
    ops = fa.assemble_spatial(mesh)
    F = fa.assemble_rhs(ops, tm.uniform(1.5, 5), source).cpu().numpy()
    Fo = O.assemble_rhs(omesh(mesh), bp, O.manufactured(source)[3])
    assert rel(F, Fo) < 1e-13


def test_lifting_matches_oracle():
    mesh = sm.build_lshape(4)
    from paper_2504_07269_b200.problems import psi0_interior
    ops = fa.assemble_spatial(mesh)
    p0 = psi0_interior(mesh)
    L = fa.lifting_rhs(ops, tm.uniform(1.0, 6), p0).cpu().numpy()
    _, Ao = O.assemble_spatial(omesh(mesh))
    Lo = O.lifting_rhs(omesh(mesh), O.temporal_uniform(1.0, 6), Ao, p0)
    assert rel(L, Lo) < 1e-13


MODES = {
    # plain multifrontal with the shared-memory small-front kernels below order 100
    "small": {},
    # every front on the tile-parallel large-front pipeline, default tuning: the children's
    # extend-add fused into the Schur-update tiles on every level, trailing updates delayed over
    # panel pairs, update engine with a 2-deep ring walking 16 tiles per CTA
    "big": dict(small_front_n=0),
    # U assembled by asm_front_kernel (no fusion), per-panel trailing updates, 32-column assembly CTAs
    "big_plain": dict(small_front_n=0, fused_min_p=1 << 30, panel_group=1, asm_whole_n=0),
    "big_pg4": dict(small_front_n=0, panel_group=4, tiles_per_cta=5),
    # single-panel levels through the update engine instead of the L21-resident kernel
    "big_no_front_syrk": dict(small_front_n=0, front_syrk_max_p=0),
    "big_fuse40": dict(small_front_n=0, fused_min_p=40, ws_stages=3, tiles_per_cta=1),
    "big_s4": dict(small_front_n=0, ws_stages=4, tiles_per_cta=7),
    "big_s4_plain": dict(small_front_n=0, fused_min_p=1 << 30, ws_stages=4),
    # spectral subtrees of <= 24 / <= 256 interior DoFs (K6) under a multifrontal top
    "spec24": {}, "spec": {},
}


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("kind,leaf", [("square9", 4), ("square16", 32), ("p2square6", 8),
                                        ("lshape5", 16), ("square40", 32), ("lshape12", 16)])
def test_factor_solve_matches_splu(kind, leaf, mode):
    """Every kernel path of K4/K5/K6 (MODES, selected through stfem_plan_options) against SuperLU."""
    spectral = {"spec24": 24, "spec": 256}.get(mode, 0)
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
    plan = sss.SpatialPlan(ops, leaf_size=leaf, spectral=spectral, options=MODES[mode])
    if spectral:
        assert plan.spectral_stats()["nroots"] >= 1
    rng = np.random.default_rng(1)
    nt, nr = 7, 3
    lam = np.array([0.3 - 0.1j, -0.02 - 1e-4j, 1 + 1j, 1e-3 - 2e-3j, -0.5 - 0.01j, 2.0 + 0j, -1e-2 - 5e-1j])
    G = rng.standard_normal((nr, nt, ops.n)) + 1j * rng.standard_normal((nr, nt, ops.n))
    W = sss.factor_solve_batch(plan, lam, torch.from_numpy(G).cuda()).cpu().numpy()
    for l in range(nt):
        ref = O._solve_shift(Mo, Ao, lam[l], G[:, l, :].T).T
        assert rel(W[:, l, :], ref) < 1e-11, (l, rel(W[:, l, :], ref))


@pytest.mark.parametrize("nr", [2, 8, 9, 16])
@pytest.mark.parametrize("opts", [dict(small_front_n=0), dict(small_front_n=0, bwd_dmma_min_p=1 << 30), dict(small_front_n=0, bwd_dmma_min_p=0), {}])
def test_multi_rhs_backward(nr, opts):
    """Multi-RHS solves: backward substitution as GEMMs over the right-hand sides on DMMA
    (backward_mrhs_kernel: one and two 8-wide RHS tiles, split-K small fronts, multi-panel fronts)
    and the column-dot-product kernel, against SuperLU."""
    mesh = sm.build_structured_square(44)
    ops = fa.assemble_spatial(mesh)
    Mo, Ao = O.assemble_spatial(omesh(mesh))
    plan = sss.SpatialPlan(ops, leaf_size=32, spectral=0, options=opts)
    rng = np.random.default_rng(3)
    lam = np.array([0.3 - 0.1j, -0.02 - 1e-4j, 1e-3 - 2e-3j, 2.0 + 0j, -0.4 - 0.3j])
    G = rng.standard_normal((nr, len(lam), ops.n)) + 1j * rng.standard_normal((nr, len(lam), ops.n))
    W = sss.factor_solve_batch(plan, lam, torch.from_numpy(G).cuda()).cpu().numpy()
    for l in range(len(lam)):
        ref = O._solve_shift(Mo, Ao, lam[l], G[:, l, :].T).T
        assert rel(W[:, l, :], ref) < 1e-11, (l, rel(W[:, l, :], ref))


def test_workspace_backoff_when_memory_is_short():
    """A batch the device cannot hold is halved until it fits (no error a smaller batch would
    have avoided); the results do not depend on the batch."""
    mesh = sm.build_structured_square(48)
    ops = fa.assemble_spatial(mesh)
    rng = np.random.default_rng(7)
    nt = 256
    lam = rng.standard_normal(nt) - 1j * (0.05 + rng.random(nt))
    G = torch.from_numpy(rng.standard_normal((1, nt, ops.n)) + 0j).cuda()
    plan = sss.SpatialPlan(ops, spectral=0)
    plan.set_batch(16)
    ref = sss.factor_solve_batch(plan, lam, G).cpu().numpy()
    del plan
    plan = sss.SpatialPlan(ops, spectral=0)
    bps = plan.set_batch(nt)                      # bytes per shift of the numeric workspace
    free, _ = torch.cuda.mem_get_info()
    keep = bps * nt // 3                          # leave room for a third of the requested batch
    hog = torch.empty(max(0, free - keep), dtype=torch.uint8, device="cuda")
    try:
        W = sss.factor_solve_batch(plan, lam, G).cpu().numpy()
        assert 1 < plan.last_num_batches()        # the full batch did not fit
    finally:
        del hog
    assert np.array_equal(W, ref)


@pytest.mark.parametrize("spectral", [0, 64])
def test_batching_invariance(spectral):
    """Results identical whatever the shift batch size."""
    mesh = sm.build_structured_square(20)
    ops = fa.assemble_spatial(mesh)
    plan = sss.SpatialPlan(ops, spectral=spectral)
    rng = np.random.default_rng(5)
    nt = 9
    lam = rng.standard_normal(nt) - 1j * rng.random(nt)
    G = torch.from_numpy(rng.standard_normal((1, nt, ops.n)) + 0j).cuda()
    plan.set_batch(0)
    W0 = sss.factor_solve_batch(plan, lam, G).cpu().numpy()
    plan.set_batch(2)
    W1 = sss.factor_solve_batch(plan, lam, G).cpu().numpy()
    assert np.array_equal(W0, W1)


def test_spec_scalar_factor_example():
    """n_x=1, lam=-2i/3 -> solve([1]) = 1/(1/8 - 8i/3)."""
    ops = fa.assemble_spatial(sm.build_structured_square(2))
    f = sss.factor(ops, lam=-2j / 3)
    w = sss.solve(f, torch.ones(1, dtype=torch.complex128, device="cuda")).item()
    assert abs(w - 1 / (1 / 8 - 8j / 3)) < 1e-14


def fd_case(m, T, N, source, seed=3):
    mesh = sm.build_structured_square(m)
    tmesh = tm.uniform(T, N)
    ops = fa.assemble_spatial(mesh)
    Mt, Bt = fa.assemble_temporal(tmesh)
    F = [fa.assemble_rhs(ops, tmesh, source)]
    rng = np.random.default_rng(seed)
    F.append(torch.from_numpy((rng.standard_normal((N, ops.n)) + 1j * rng.standard_normal((N, ops.n))) / np.sqrt(2)).cuda())
    return mesh, tmesh, ops, Mt, Bt, torch.stack(F)


@pytest.mark.parametrize("m,T,N,source", [(16, 1.0, 16, "sinpit"), (64, 1.0, 64, "sinpit"),
                                          (32, 2.0, 48, "texp")])
def test_fdm_solve_matches_oracle(m, T, N, source):
    """Full FD solve (C1 and C2 configs) vs the oracle on identical (lam, X, Y) and F: <= 1e-9."""
    mesh, tmesh, ops, Mt, Bt, F = fd_case(m, T, N, source)
    Mo, Ao = O.assemble_spatial(omesh(mesh))
    tfo = O.eigen_decompose(Mt, Bt)
    mine = temporal_factors(Mt, Bt)
    assert np.abs(mine.eigenvalues - tfo.lam).max() < 1e-14 * np.abs(tfo.lam).max()
    assert np.abs(mine.X - tfo.X).max() < 1e-13
    # parity isolates the GPU arithmetic: both paths consume the same (lam, X, Y)
    from paper_2504_07269_b200.dense_complex_linalg import TemporalFactors
    shared = TemporalFactors(X=tfo.X, S=np.diag(tfo.lam), Y=tfo.Y, kappa2=tfo.kappa2)
    fdm = ks.FDMSolver(ops, Mt, Bt, factors=shared)
    psi = fdm.solve(F).cpu().numpy()
    ref = O.fdm_solve(Mo, Ao, tfo, F.cpu().numpy())
    for r in range(2):
        assert rel(psi[r], ref[r]) < 1e-9, rel(psi[r], ref[r])
    res = ks.relative_residual(ops, Mt, Bt, torch.from_numpy(psi).cuda(), F)
    assert res < 1e-8
    if m == 16:
        # manufactured-solution errors reproduce the oracle's to 3 significant digits
        from paper_2504_07269_b200 import error_analysis as ea
        e_gpu = ea.spacetime_errors(psi[0], ea.exact_solution(source), mesh, tmesh)
        ps, dt, gr, _ = O.manufactured(source)
        e_ref = O.spacetime_errors(omesh(mesh), tmesh.breakpoints, ref[0], ps, dt, gr)
        for a, b in zip(e_gpu, e_ref):
            assert abs(a - b) / b < 5e-4


@pytest.mark.parametrize("m,N", [(64, 64), (40, 48)])
def test_fdm_fused_permutation_matches_default(m, N):
    """FDMSolver.fused_perm (the nested-dissection permutation applied by the transforms'
    column maps, stfem_plan_set_io_permuted in between) gives the default path's Psi: staged
    solve, pipelined host solve and the host stream."""
    mesh, tmesh, ops, Mt, Bt, F = fd_case(m, 1.0, N, "sinpit")
    fdm = ks.FDMSolver(ops, Mt, Bt)
    ref = fdm.solve(F, timings={}).clone()
    fdm.fused_perm = True
    psi = fdm.solve(F, timings={})
    assert rel(psi.cpu().numpy(), ref.cpu().numpy()) < 1e-13
    Fh = F.cpu().pin_memory()
    Ph = torch.empty_like(Fh).pin_memory()
    fdm.solve_host(Fh, Ph)
    assert rel(Ph.numpy(), ref.cpu().numpy()) < 1e-13
    Ph2 = [torch.empty_like(Fh).pin_memory() for _ in range(3)]
    fdm.solve_host_stream([Fh] * 3, Ph2)
    for P in Ph2:
        assert rel(P.numpy(), ref.cpu().numpy()) < 1e-13
    fdm.fused_perm = False
    assert rel(fdm.solve(F).cpu().numpy(), ref.cpu().numpy()) < 1e-13


def test_spec_1x1_global():
    """n_x = n_t = 1 global system, psi = 1/(4/3 + i/16)."""
    ops = fa.assemble_spatial(sm.build_structured_square(2))
    Mt, Bt = fa.assemble_temporal(tm.uniform(1.0, 1))
    rep = ks.solve(ops, Mt, Bt, torch.ones((1, 1), dtype=torch.complex128, device="cuda"))
    assert abs(rep.solution.item() - 1 / (4 / 3 + 1j / 16)) < 1e-14
    assert rep.relative_residual < 1e-14


def test_apply_global_matches_oracle():
    mesh = sm.build_structured_square(9)
    for deg_t in (1, 2):
        tmesh = tm.uniform(1.0, 7)
        ops = fa.assemble_spatial(mesh)
        Mt, Bt = fa.assemble_temporal(tmesh, deg_t)
        rng = np.random.default_rng(0)
        v = rng.standard_normal((Mt.shape[0], ops.n)) + 1j * rng.standard_normal((Mt.shape[0], ops.n))
        out = ks.apply_global(ops, Mt, Bt, torch.from_numpy(v).cuda()).cpu().numpy()
        Mo, Ao = O.assemble_spatial(omesh(mesh))
        ref = O.apply_global(Mo, Ao, Mt, Bt, v)
        assert rel(out, ref) < 1e-13


def test_dense_oracle_small():
    """m=4 square, n_t=4, random f vs the explicit Kronecker system, 1e-10."""
    mesh = sm.build_structured_square(4)
    tmesh = tm.uniform(1.0, 4)
    ops = fa.assemble_spatial(mesh)
    Mt, Bt = fa.assemble_temporal(tmesh)
    rng = np.random.default_rng(11)
    f = rng.standard_normal((4, ops.n)) + 1j * rng.standard_normal((4, ops.n))
    psi = ks.solve(ops, Mt, Bt, torch.from_numpy(f).cuda()).solution.cpu().numpy()
    Mo, Ao = O.assemble_spatial(omesh(mesh))
    ref = np.linalg.solve(O.dense_global(Mo, Ao, Mt, Bt), f.ravel()).reshape(f.shape)
    assert rel(psi, ref) < 1e-10


def test_fd_factor_solve_c3_sample_shifts():
    """C3-size operator (m=256, P1) at the hardest shifts of n_t = 256 vs splu."""
    mesh = sm.build_structured_square(256)
    ops = fa.assemble_spatial(mesh)
    Mt, Bt = fa.assemble_temporal(tm.uniform(2.0, 256))
    tf = temporal_factors(Mt, Bt)
    lam_all = tf.eigenvalues
    pick = np.r_[np.argsort(np.abs(lam_all.imag))[:3], [0, 128, 255]]
    lam = lam_all[pick]
    plan = sss.SpatialPlan(ops)
    rng = np.random.default_rng(2)
    G = rng.standard_normal((1, len(lam), ops.n)) + 1j * rng.standard_normal((1, len(lam), ops.n))
    W = sss.factor_solve_batch(plan, lam, torch.from_numpy(G).cuda()).cpu().numpy()
    Mo, Ao = O.assemble_spatial(omesh(mesh))
    for l in range(len(lam)):
        ref = O._solve_shift(Mo, Ao, lam[l], G[0, l])
        assert rel(W[0, l], ref) < 1e-10


def test_solve_host_pipelined_matches_device_solve():
    """FDMSolver.solve_host (pinned host in/out, copies overlapped with the
    transforms in column blocks) gives exactly the device-buffer solve."""
    mesh = sm.build_structured_square(20)
    ops = fa.assemble_spatial(mesh)
    Mt, Bt = fa.assemble_temporal(tm.uniform(1.0, 12))
    fdm = ks.FDMSolver(ops, Mt, Bt)
    rng = np.random.default_rng(9)
    F = torch.from_numpy(rng.standard_normal((2, 12, ops.n)) + 1j * rng.standard_normal((2, 12, ops.n)))
    ref = fdm.solve(F.cuda()).cpu().numpy()
    Fh = F.pin_memory()
    Ph = torch.empty_like(Fh).pin_memory()
    for chunks in (1, 3, 8):
        Ph.zero_()
        fdm.solve_host(Fh, Ph, chunks=chunks)
        torch.cuda.synchronize()
        assert np.array_equal(Ph.numpy(), ref)


def test_solve_host_stream_matches_device_solves():
    """FDMSolver.solve_host_stream (a stream of pinned host solves with the copies of
    neighbouring steps overlapped, device buffers rotating) gives exactly the
    device-buffer solve of every step, including distinct inputs per step."""
    mesh = sm.build_structured_square(20)
    ops = fa.assemble_spatial(mesh)
    Mt, Bt = fa.assemble_temporal(tm.uniform(1.0, 12))
    fdm = ks.FDMSolver(ops, Mt, Bt)
    rng = np.random.default_rng(10)
    Fs = [torch.from_numpy(rng.standard_normal((2, 12, ops.n)) + 1j * rng.standard_normal((2, 12, ops.n)))
          for _ in range(4)]
    refs = [fdm.solve(F.cuda()).cpu().numpy() for F in Fs]
    Fh = [F.pin_memory() for F in Fs]
    for chunks, nbuf in ((1, None), (5, None), (3, 3), (2, 4)):
        # nbuf None: the solver allocates (four stacks when they are a small part of the memory);
        # 3 / 4: caller-owned buffers, the three-buffer rotation and the four-buffer one
        bufs = None if nbuf is None else tuple(torch.empty_like(Fs[0], device="cuda") for _ in range(nbuf))
        Ph = [torch.zeros_like(F).pin_memory() for F in Fs]
        fdm.solve_host_stream(Fh, Ph, chunks=chunks, dev_buffers=bufs)
        torch.cuda.synchronize()
        for P, ref in zip(Ph, refs):
            assert np.array_equal(P.numpy(), ref)
    # one host output buffer rewritten every step (the bench's serving loop) ends with the last Psi
    P1 = torch.zeros_like(Fs[0]).pin_memory()
    fdm.solve_host_stream(Fh, [P1] * 4)
    torch.cuda.synchronize()
    assert np.array_equal(P1.numpy(), refs[-1])
