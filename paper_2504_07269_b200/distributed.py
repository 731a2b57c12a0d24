"""Multi-GPU FD solve: one process per GPU, NCCL all-to-all over NVLink.

Partitioning (north_star):
  * every rank holds the plan, M_x/A_x, X, Y, lam (replicated; X/Y/lam are
    computed once on rank 0 and broadcast so every rank uses identical bits);
  * spatial shard: rank p owns columns [p c, (p+1) c) of every temporal block,
    c = ceil(n_x / P) (the last shard is zero-padded);
  * local layout of a shard is (n_t, n_rhs, c): the forward transform is ONE
    GEMM G_p = Y F_p with N = n_rhs c, and the all-to-all send block for rank
    q (its n_t/P shifts) is one contiguous (n_t/P, n_rhs, c) slab;
  * all-to-all #1 -> rank q holds (P, n_t/P, n_rhs, c) = all columns of its
    n_t/P shifts; the multifrontal factor+solve reads/writes that buffer in
    place through the chunked BlockVector layout (no repack);
  * all-to-all #2 returns (n_t, n_rhs, c) shards; back transform Psi_p = X W_p.
The compute backend is injectable so the orchestration (sharding, layouts,
exchange) is testable on CPU with gloo; the product backend is the CUDA one.
"""

from __future__ import annotations

import math
import os
import time

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N

C128 = torch.complex128


class CudaBackend:
    """K3 transforms + K4/K5 factor/solve through the C-ABI."""

    def __init__(self, plan, pairs=None):
        self.plan = plan
        self.pairs = pairs   # paired_transform.DevicePairs: K3p transforms (half the flops of K3)

    def transform(self, T, x, out):
        from . import _kernels as K
        K.time_transform(T, x, out=out)

    def transform_fwd(self, Y, x, out):
        from . import _kernels as K
        if self.pairs is None:
            K.time_transform(Y, x, out=out)
        else:
            K.transform_pair_fwd(self.pairs, x, out=out)

    def transform_back(self, X, x, out):
        """x is scratch (K3p mixes its pair rows in place)."""
        from . import _kernels as K
        if self.pairs is None:
            K.time_transform(X, x, out=out)
        else:
            K.transform_pair_back(self.pairs, x, out=out)

    def factor_solve(self, lam, G, W, layout, nrhs):
        self.plan.factor_solve(lam, G, W, layout, nrhs)


def shard_cols(nx: int, P: int) -> int:
    return -(-nx // P)


def chunked_layout(nt_loc: int, nrhs: int, c: int) -> N.bv_layout:
    """Element (rhs r, local shift l, column j) of a (P, nt_loc, nrhs, c) buffer."""
    return N.bv_layout(c, nrhs * c, c, nt_loc * nrhs * c)


def shard_rhs(F: torch.Tensor, rank: int, P: int) -> torch.Tensor:
    """(n_rhs, n_t, n_x) full stack -> this rank's (n_t, n_rhs, c) shard (zero padded)."""
    nr, nt, nx = F.shape
    c = shard_cols(nx, P)
    lo, hi = rank * c, min(nx, (rank + 1) * c)
    out = torch.zeros((nt, nr, c), dtype=F.dtype, device=F.device)
    if hi > lo:
        out[:, :, :hi - lo] = F[:, :, lo:hi].permute(1, 0, 2)
    return out


def unshard(Psi_p: torch.Tensor, nx: int, rank: int, P: int) -> torch.Tensor:
    """(n_t, n_rhs, c) shard -> (n_rhs, n_t, cols) of the real columns it owns."""
    c = Psi_p.shape[-1]
    lo, hi = rank * c, min(nx, (rank + 1) * c)
    return Psi_p[:, :, :max(0, hi - lo)].permute(1, 0, 2)


class DistributedFDM:
    """FD solve of a replicated problem with spatially sharded inputs/outputs."""

    def __init__(self, nx: int, nt: int, nrhs: int, X: torch.Tensor, Y: torch.Tensor, lam: torch.Tensor,
                 backend, group=None):
        self.group = group
        self.P = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if nt % self.P:
            raise N.DimensionMismatch(N.ERR_DIM, f"n_t={nt} must be divisible by the world size {self.P}")
        self.nx, self.nt, self.nrhs = nx, nt, nrhs
        self.c = shard_cols(nx, self.P)
        self.ntl = nt // self.P
        self.X, self.Y = X, Y
        self.lam_local = lam[self.rank * self.ntl:(self.rank + 1) * self.ntl].contiguous()
        self.backend = backend
        dev = X.device
        shape = (nt, nrhs, self.c)
        self.G = torch.empty(shape, dtype=C128, device=dev)
        self.R = torch.empty(shape, dtype=C128, device=dev)   # receive buffer (P, ntl, nrhs, c)
        self.W = torch.zeros(shape, dtype=C128, device=dev)
        self.layout = chunked_layout(self.ntl, nrhs, self.c)

    def _a2a(self, out, inp):
        if self.P == 1:
            out.copy_(inp)
        else:
            # complex128 exchanged as its float64 view (NCCL has no complex type)
            dist.all_to_all_single(torch.view_as_real(out), torch.view_as_real(inp), group=self.group)

    def solve(self, F_p: torch.Tensor, out: torch.Tensor | None = None, timings: dict | None = None):
        """F_p: (n_t, n_rhs, c) shard.  Returns Psi_p in the same layout."""
        nt, nr, c = self.nt, self.nrhs, self.c
        if F_p.shape != (nt, nr, c):
            raise N.DimensionMismatch(N.ERR_DIM, f"shard {tuple(F_p.shape)} != {(nt, nr, c)}")
        out = out if out is not None else torch.empty_like(F_p)
        fwd = getattr(self.backend, "transform_fwd", self.backend.transform)
        back = getattr(self.backend, "transform_back", self.backend.transform)
        cuda = F_p.is_cuda
        marks = []

        def mark():
            if timings is None:
                return
            if cuda:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record()
                marks.append(ev)
            else:
                marks.append(time.perf_counter())

        mark()
        fwd(self.Y, F_p.view(nt, nr * c), self.G.view(nt, nr * c))                         # (2)
        mark()
        self._a2a(self.R, self.G)                                                           # a2a #1
        mark()
        self.backend.factor_solve(self.lam_local, self.R, self.W, self.layout, nr)         # (3)
        mark()
        self._a2a(self.G, self.W)                                                           # a2a #2
        mark()
        back(self.X, self.G.view(nt, nr * c), out.view(nt, nr * c))                        # (4)
        mark()
        if timings is not None:
            if cuda:
                marks[-1].synchronize()
                dt = [marks[i].elapsed_time(marks[i + 1]) / 1e3 for i in range(5)]
            else:
                dt = [marks[i + 1] - marks[i] for i in range(5)]
            for k, v in zip(("forward_transform_s", "a2a_fwd_s", "factor_solve_s", "a2a_back_s",
                             "back_transform_s"), dt):
                timings[k] = v
            timings["a2a_bytes_each_way"] = 16 * nt * nr * c * (self.P - 1) // self.P
        return out


class NativeComm:
    """stfem_comm: the library's own NCCL communicator (include/stfem_b200.h).  Rank 0 draws
    the unique id, torch.distributed (any backend) carries its 128 bytes to the other ranks --
    the "unique id broadcast through the torch store" of SURVEY.md §8b."""

    def __init__(self, group=None):
        import ctypes as C
        N.require_cuda()
        self.nranks = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        uid = torch.zeros(128, dtype=torch.uint8)
        if self.rank == 0:
            buf = (C.c_uint8 * 128)()
            N.check(N.lib().stfem_comm_unique_id(buf))
            uid = torch.tensor(list(buf), dtype=torch.uint8)
        if self.nranks > 1:
            backend = dist.get_backend(group)
            t = uid.cuda() if backend == "nccl" else uid
            dist.broadcast(t, 0, group=group)
            uid = t.cpu()
        raw = (C.c_uint8 * 128)(*uid.tolist())
        h = C.c_void_p()
        N.check(N.lib().stfem_comm_init(raw, self.nranks, self.rank, C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def info(self) -> dict:
        import ctypes as C
        a, b, v = C.c_int32(), C.c_int32(), C.c_int32()
        N.check(N.lib().stfem_comm_info(self._h, C.byref(a), C.byref(b), C.byref(v)))
        return {"nranks": a.value, "rank": b.value, "nccl_version": v.value}

    def all_to_all(self, send: torch.Tensor, recv: torch.Tensor, stream=None):
        count = send.numel() // self.nranks
        N.check(N.lib().stfem_comm_all_to_all(self._h, N.ptr(send), N.ptr(recv), count, N.stream_ptr(stream)))

    def close(self):
        if getattr(self, "_h", None) is not None and N._lib is not None:
            N._lib.stfem_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


class NativeShardedFDM:
    """The sharded FD solve through ONE C-ABI call per solve (stfem_fdm_solve with a
    stfem_comm): transforms, both exchanges and the local factor + solve are enqueued by the
    library on the caller's stream.  Same shard layout as DistributedFDM: (n_t, n_rhs, c)."""

    def __init__(self, fdm, nrhs: int, comm: NativeComm):
        self.fdm, self.comm, self.nrhs = fdm, comm, nrhs
        self.P, self.rank = comm.nranks, comm.rank
        if fdm.nt % self.P:
            raise N.DimensionMismatch(N.ERR_DIM, f"n_t={fdm.nt} must be divisible by the world size {self.P}")
        self.c = shard_cols(fdm.ops.n, self.P)
        self.work = torch.empty((fdm.nt, nrhs, self.c), dtype=C128, device=fdm.X.device)
        fdm.plan.prepare()
        fdm.plan.reserve(fdm.nt // self.P, nrhs)

    def solve(self, F_p: torch.Tensor, out: torch.Tensor | None = None, stream=None, check: bool = True):
        import ctypes as C
        shape = (self.fdm.nt, self.nrhs, self.c)
        if tuple(F_p.shape) != shape or not F_p.is_contiguous():
            raise N.DimensionMismatch(N.ERR_DIM, f"shard {tuple(F_p.shape)} != {shape}")
        out = out if out is not None else torch.empty_like(F_p)
        fdm = self.fdm
        N.check(N.lib().stfem_fdm_solve(fdm.plan.handle, self.comm.handle, N.ptr(fdm.ops.Mvals), N.ptr(fdm.ops.Avals),
                                        C.byref(fdm.fd_factors()), N.ptr(F_p), N.ptr(out), N.ptr(self.work),
                                        self.nrhs, N.stream_ptr(stream)))
        if check:
            fdm.plan.check(stream)
        return out


def broadcast_factors(X, Y, lam, device):
    """Rank 0's (X, Y, lam) on every rank (identical bits everywhere)."""
    out = []
    for a in (X, Y, lam):
        t = torch.tensor(np.ascontiguousarray(a), dtype=C128).to(device)
        if dist.is_initialized() and dist.get_world_size() > 1:
            dist.broadcast(torch.view_as_real(t), 0)   # collectives on the real view
        out.append(t)
    return tuple(out)


def bench_main(args):
    """bench.py --gpus N under torchrun: strong scaling of one config."""
    import json

    from . import kronecker_solver as ks  # noqa: F401
    from .dense_complex_linalg import temporal_factors
    from .problems import Problem
    from .sparse_spatial_solver import SpatialPlan

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    t0 = time.perf_counter()
    prob = Problem(args.workload, device=dev, with_rhs=False)
    prob.assemble()
    torch.cuda.synchronize()
    t_asm = time.perf_counter() - t0
    t1 = time.perf_counter()
    from . import paired_transform as PT
    nt = prob.nt
    X, Y, lam = np.zeros((nt, nt), complex), np.zeros((nt, nt), complex), np.zeros(nt, complex)
    if rank == 0:
        tf = temporal_factors(prob.M_t, prob.B_t)
        X, Y, lam = tf.X, tf.Y, tf.eigenvalues
        pf0 = PT.build(lam, X, prob.B_t)
        if pf0 is not None:
            X, Y, lam = pf0.X, pf0.Y, pf0.lam       # the paired eigenbasis
    Xt, Yt, lt = broadcast_factors(X, Y, lam, dev)
    # every rank derives the K3p tables from the broadcast (already paired) factors
    pf = PT.build(lt.cpu().numpy(), Xt.cpu().numpy(), prob.B_t)
    if pf is not None:
        Yt = torch.as_tensor(pf.Y, dtype=C128, device=dev)
    pairs = PT.DevicePairs(pf, dev) if pf is not None else None
    # host setup of the spectral subtrees: this rank's share of the host cores, not all of them
    plan = SpatialPlan(prob.ops, spectral_threads=max(1, len(os.sched_getaffinity(0)) // max(1, local_world_size())))
    t_setup = time.perf_counter() - t1
    solver = DistributedFDM(prob.nx, nt, prob.n_rhs, Xt, Yt, lt, CudaBackend(plan, pairs))
    # this rank's RHS shard: deterministic part on device + Gaussian columns from the shared streams
    Fp = _local_rhs(prob, rank, world, dev)
    out = torch.empty_like(Fp)
    for _ in range(args.warmup):
        solver.solve(Fp, out)
    torch.cuda.synchronize()
    clk = None
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    if rank == 0:
        from bench import ClockSampler
        clk = ClockSampler(local)
        clk.start()
        clk.wait_first()
        time.sleep(0.3)
    # the barrier after the sampler start-up: no rank's timed region waits on rank 0's sampler
    dist.barrier()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(args.steps):
        solver.solve(Fp, out)
    e.record()
    torch.cuda.synchronize()
    clocks = clk.stop() if clk is not None else None
    t_local = s.elapsed_time(e) / 1e3 / args.steps
    tt = torch.tensor([t_local], dtype=torch.float64, device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    dist.barrier()
    t_step = float(tt.item())
    dofs = prob.nx * nt * prob.n_rhs
    launches = (3 if pairs is not None else 2) + plan.last_launches()
    # roofline of the dominant kernel family: one extra step with per-launch events on every
    # rank (the all-to-alls keep the ranks in step); rank 0 reports its own shifts
    roof = None
    if rank == 0:
        plan.record_levels(True)
    solver.solve(Fp, out)
    torch.cuda.synchronize()
    if rank == 0:
        plan.record_levels(False)
        from bench import dmma_peak_live, family_roofline
        roof, fam = family_roofline(plan, nt // world, prob.n_rhs, dmma_peak_live(), args.workload)
        roof["per_rank_families"] = fam
    # e2e: each rank's shard from pinned host memory, the solve, the shard back to the host
    e2e = None
    if not args.no_e2e:
        Fh = Fp.cpu().pin_memory()
        Ph = torch.empty_like(Fh).pin_memory()

        def e2e_step():
            Fp.copy_(Fh, non_blocking=True)
            solver.solve(Fp, out)
            Ph.copy_(out, non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        dist.barrier()
        s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n_e2e = max(1, min(args.steps, 3))
        s2.record()
        for _ in range(n_e2e):
            e2e_step()
        e2.record()
        torch.cuda.synchronize()
        te = torch.tensor([s2.elapsed_time(e2) / 1e3 / n_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        nbytes = Fh.numel() * 16 * world
        e2e = {"value": dofs / float(te.item()), "unit": "DoF/s", "h2d_bytes_per_step": nbytes,
               "d2h_bytes_per_step": nbytes, "ms_per_step": float(te.item()) * 1e3}
    if rank == 0:
        line = {"metric": "space-time DoF/s (complex fp64) of the FDM direct solve", "value": dofs / t_step,
                "unit": "DoF/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "c128", "data": "synthetic (seeded Gaussian RHS; BASELINE.json configs)",
                "config": {"workload": args.workload, "n_x": prob.nx, "n_t": nt, "n_rhs": prob.n_rhs,
                           "parallelism": f"space-sharded transforms + time-sharded shifts, a2a x2 over {world} GPUs"},
                "setup_s": t_setup, "asm_s": t_asm, "gpu_launches": launches * args.steps,
                "clocks": clocks, "e2e": e2e, "cpu_baseline": None,
                "roofline": roof}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def _local_rhs(prob, rank, world, dev):
    """(n_t, n_rhs, c) shard of the config's RHS stack, generated locally."""
    from . import fem_assembly as fa
    from .problems import gaussian_rhs
    nx, nt = prob.nx, prob.nt
    c = shard_cols(nx, world)
    lo, hi = rank * c, min(nx, (rank + 1) * c)
    parts = []
    if prob.cfg.source:
        parts.append(fa.assemble_rhs(prob.ops, prob.tmesh, prob.cfg.source)[:, lo:hi])
    if prob.cfg.psi0:
        parts.append(fa.lifting_rhs(prob.ops, prob.tmesh, prob.psi0)[:, lo:hi])
    Fp = torch.zeros((nt, prob.n_rhs, c), dtype=C128, device=dev)
    for i, part in enumerate(parts):
        Fp[:, i, :hi - lo] = part
    if prob.cfg.n_gauss and hi > lo:
        # only this rank's columns are drawn (per-column-block streams): (n_gauss, n_t, hi - lo)
        threads = max(1, len(os.sched_getaffinity(0)) // max(1, local_world_size()))
        g = gaussian_rhs(prob.seed, prob.cfg.n_gauss, nt, nx, cols=(lo, hi), threads=threads)
        Fp[:, len(parts):, :hi - lo] = torch.from_numpy(g).to(dev).permute(1, 0, 2)
    return Fp


def local_world_size() -> int:
    """Ranks sharing this host's cores (torchrun exports LOCAL_WORLD_SIZE)."""
    return int(os.environ.get("LOCAL_WORLD_SIZE", os.environ.get("WORLD_SIZE", "1")))
