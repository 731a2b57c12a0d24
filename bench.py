#!/usr/bin/env python
"""Benchmark: space-time DoF/s (complex fp64) of the FDM direct solve.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C4] [--impl ours|reference]

One step = one FD solve of the workload's RHS stack: forward time transform
(K3p, DMMA), n_t batched multifrontal factor+solve (K4/K5), back transform (K3p)
(+ the two all-to-alls when N > 1).  `value` = n_x * n_t * n_rhs / t_step
(whole job), inputs resident in HBM (each input array of the big configs is larger
than L2; C1/C2 rewrite a 256 MB buffer before every timed step).  `e2e` = the same metric through the public API with the
pinned host->device copy of F and the device->host copy of Psi inside the
timed region.  Host setup (temporal eigendecomposition + symbolic analysis) is
reported separately as setup_s, assembly as asm_s.

`--impl reference` times the reference's FDM path on the host: the CPU
restatement in oracle/ (SuperLU per shift via scipy, numpy transforms; the
reference ships no runnable FDM code), built from oracle/ alone (no product
code is imported or mapped), all host threads, on a bounded sample of shifts
per step (disjoint across steps); rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_WORKLOAD = "C4"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default=os.environ.get("STFEM_WORKLOAD", DEFAULT_WORKLOAD))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sample-shifts", type=int, default=0)
    ap.add_argument("--proxy-ranks", type=int, default=0,
                    help="one-GPU proxy of a P-rank run: time ONE rank's share (transforms on n_x/P columns, "
                         "n_t/P shifts, the exchange volume) and print the predicted P-GPU time")
    ap.add_argument("--plan-opt", action="append", default=[],
                    help="stfem_plan_options field name=value (repeatable; A/B runs of a tuning knob)")
    ap.add_argument("--variant", default="fd", choices=["fd", "bs"],
                    help="fd: fast diagonalization (the headline path); bs: Bartels-Stewart sweep (SPEC.md:377)")
    return ap.parse_args()


# ----------------------------------------------------------------------------
# clocks sampled during the timed region
# ----------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (FileNotFoundError, OSError):
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def wait_first(self, timeout=10.0):
        """Block until nvidia-smi has produced its first sample: its NVML start-up stalls the
        driver for a moment and must not land inside a short timed region (C2 steps are ~1 ms)."""
        t0 = time.time()
        while self.proc is not None and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.02)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


# ----------------------------------------------------------------------------
# reference arm: the oracle's CPU FDM path (numpy / scipy only -- it imports nothing from
# the product package and maps none of its native code) on a bounded sample of shifts
# ----------------------------------------------------------------------------
L2_BYTES = 126 * 2 ** 20

# workload -> (oracle mesh builder, degree_x, degree_t, T, N, deterministic RHS, Gaussian RHS)
ORACLE_CONFIGS = {
    "C1": ("square:16", 1, 1, 1.0, 16, 1, 1),
    "C2": ("square:64", 1, 1, 1.0, 64, 1, 1),
    "C3": ("square:256", 1, 1, 2.0, 256, 1, 1),
    "C4": ("p2square:256", 2, 2, 1.0, 512, 0, 1),
    "C5": ("lshape:256", 1, 1, 1.0, 1024, 1, 8),
}


def config_dict(workload, nx, nt, nrhs, world=1):
    """The `config` object of the JSON line: identical in both arms for one workload."""
    big = 16 * nx * nt * nrhs > L2_BYTES
    return {"workload": workload, "n_x": int(nx), "n_t": int(nt), "n_rhs": int(nrhs), "dofs_per_rhs": int(nx * nt),
            "parallelism": "single" if world == 1 else f"space/time sharded x{world}",
            "l2": ("inputs larger than L2 (F, G, Psi each > 126 MB); no flush" if big else
                   "inputs fit in L2: a 256 MB buffer is rewritten before every timed step (outside the events)")}


class OracleProblem:
    """A BASELINE.json config built from oracle/ alone (meshes, operators, temporal pencil)."""

    def __init__(self, workload):
        from oracle import stfem_oracle as O
        spec, dx, dt, T, N, ndet, ngauss = ORACLE_CONFIGS[workload]
        kind, arg = spec.split(":")
        if kind == "square":
            mesh, els = O.square_mesh(int(arg)), None
        elif kind == "p2square":
            mesh, els = O.refine_mesh(O.square_mesh(int(arg)))
        else:
            mesh, els = O.lshape_mesh(int(arg)), None
        els = mesh.elements if els is None else els
        self.Mx, self.Ax = O.assemble_spatial_vec(mesh.vertices, els, mesh.interior_dof, dx)
        self.nx = self.Mx.shape[0]
        bp = O.temporal_uniform(T, N)
        self.M_t, self.B_t = O.assemble_temporal(bp, dt)
        self.nt = self.M_t.shape[0]
        self.n_rhs = ndet + ngauss
        self.coords = O.dof_coordinates(mesh.vertices, mesh.interior_dof)
        self.tf = O.eigen_decompose(self.M_t, self.B_t)
        self.perm = O.nd_ordering(self.Ax, self.coords, leaf=16)
        self.pair = O.permuted_csc_pair(self.Mx, self.Ax, self.perm)


def cpu_fdm_sample(op, F, shifts, pool, mode="nd"):
    """Time the CPU FD path restricted to `shifts`: G_s = Y_s F (BLAS zgemm), per-shift
    SuperLU factor + solve on the worker pool (mode "nd": shared nested-dissection
    ordering, no pivoting -- the fastest SuperLU configuration; "mmd": minimum-degree
    ordering + partial pivoting), Psi += X_s W_s.  Returns seconds."""
    tf = op.tf
    t0 = time.perf_counter()
    Ys = np.ascontiguousarray(tf.Y[shifts])
    G = np.stack([Ys @ F[r] for r in range(F.shape[0])])      # (n_rhs, k, n_x)
    sols = pool.solve(tf.lam[shifts], [np.ascontiguousarray(G[:, i, :].T) for i in range(len(shifts))], mode)
    W = np.stack(sols, axis=0).transpose(2, 0, 1)             # (n_rhs, k, n_x)
    Xs = np.ascontiguousarray(tf.X[:, shifts])
    _ = [Xs @ np.ascontiguousarray(W[r]) for r in range(W.shape[0])]   # back-transform contribution
    return time.perf_counter() - t0


def complex_gaussian(seed, shape):
    rng = np.random.default_rng(seed)
    F = np.empty(shape, dtype=complex)
    F.real = rng.standard_normal(shape)
    F.imag = rng.standard_normal(shape)
    F *= 1 / np.sqrt(2)
    return F


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import stfem_oracle as O
    op = OracleProblem(args.workload)
    threads = O.cpu_threads()
    # bounded sample: every step solves its own, disjoint set of shifts (a seeded permutation
    # walked step by step), one wave of the host workers per step by default
    k = min(args.sample_shifts or threads, op.nt)
    threads = min(threads, k)
    pool = O.ShiftPool(op.Mx, op.Ax, op.perm, threads)
    F = complex_gaussian(0, (op.n_rhs, op.nt, op.nx))
    order = np.random.default_rng(1).permutation(op.nt)
    nsteps = args.warmup + args.steps
    samples = [np.sort(order[(i * k + np.arange(k)) % op.nt]) for i in range(nsteps)]
    for s in samples[:args.warmup]:
        cpu_fdm_sample(op, F, s, pool)
    times = [cpu_fdm_sample(op, F, s, pool) for s in samples[args.warmup:]]
    t = max(statistics.mean(times), 1e-12)
    dofs = op.nx * k * op.n_rhs
    val = dofs / t
    # the same sample size through the pivoting mode (one step), for reference
    t_mmd = cpu_fdm_sample(op, F, samples[-1], pool, mode="mmd")
    pool.close()
    distinct = len(np.unique(np.concatenate(samples[args.warmup:])))
    sample = (f"{k} of {op.nt} shifts per step, disjoint across steps ({distinct} distinct shifts solved in the "
              f"timed region = {100.0 * distinct / op.nt:.0f}% of the workload), sampled transforms + SuperLU "
              f"factor/solve per shift, {op.n_rhs} RHS, complex Gaussian F")
    line = {"metric": "space-time DoF/s (complex fp64) of the FDM direct solve", "value": val, "unit": "DoF/s",
            "impl": "reference", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "c128", "data": "synthetic (seeded Gaussian RHS; BASELINE.json configs)",
            "config": config_dict(args.workload, op.nx, op.nt, op.n_rhs),
            "cpu_baseline": {"value": val, "unit": "DoF/s", "cores": threads, "kind": "port", "sample": sample,
                             "parallelism": f"{threads} worker processes, one shift each, 1 BLAS thread per worker",
                             "cpu_model": O.cpu_model(), "host_cores_visible": O.cpu_threads(),
                             "superlu_mode": "shared nested-dissection ordering, no pivoting (fastest; SURVEY App. A)",
                             "pivoting_mode_value": dofs / t_mmd,
                             "pivoting_mode": "MMD(A^T+A) ordering + partial pivoting, one step of the same size"},
            "e2e": {"value": val, "unit": "DoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------
def dmma_peak_live():
    """FP64 tensor-pipe peak measured now on this GPU (register-only DMMA loop)."""
    import ctypes as C
    import torch
    from paper_2504_07269_b200 import _native as N
    sm = torch.cuda.get_device_properties(0).multi_processor_count
    sink = torch.zeros(256, dtype=torch.float64, device="cuda")
    fl = C.c_double()
    best = 0.0
    for it in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        N.check(N.lib().stfem_probe_launch(0, sm * 2, 20000, N.ptr(sink), C.byref(fl), N.stream_ptr()))
        e.record()
        e.synchronize()
        best = max(best, fl.value / (s.elapsed_time(e) / 1e3) / 1e12)
    return best


def hbm_peak():
    """(GB/s, source): MEASURED_PEAKS.json's copy bandwidth, else the profiling recipe's fallback."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            v = float(json.load(f)["hbm_gbs"])
        return v, "MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback: 6.65 TB/s from B200_PROFILING.md (MEASURED_PEAKS.json absent)"


FAMILY_NAMES = {"spectral": "spectral_kernel (K6 spectral subtrees, DMMA)",
                "assembly": "asm_front_kernel (front assembly, HBM)",
                "diag": "diag_kernel (diagonal blocks, FP64)",
                "trsm": "trsm_kernel (panel TRSM, FP64)",
                "panel_update": "panel_ws_kernel (trailing pivot columns, warp-specialised TMA-fed update engine, DMMA)",
                "syrk": "syrk_ws_kernel (Schur updates U = sum children - L21 L21^T on the warp-specialised TMA-fed "
                        "update engine; single-panel levels: syrk_front_kernel, L21 resident in shared memory; DMMA, "
                        "3M complex product)",
                "backward": "backward kernels (HBM)",
                "small_factor": "factor_small_kernel (shared-memory fronts)"}


def family_roofline(plan, nshift, nrhs, peak, workload, t_tr=None, flops_tr=None):
    """(roofline of the dominant kernel family, per-family table) from the plan's last
    recorded factor_solve (record_levels) over `nshift` shifts; the transforms join the
    table when their time t_tr (s) and flops are given."""
    rep = plan.kernel_report()
    if plan.spectral is not None:
        ss = plan.spectral_stats()
        rep["spectral"] = (rep["spectral"][0], ss["flops_u"] + nrhs * ss["flops_rhs"], rep["spectral"][2])
    fam = {}
    for k, (ms, fl, nl) in rep.items():
        if nl == 0:
            continue
        tf = fl * nshift / (ms / 1e3) / 1e12 if ms > 0 else 0.0
        fam[k] = {"ms": ms, "launches": nl, "tflops": tf, "frac_dmma": tf / peak}
    if t_tr:
        fam["transform"] = {"ms": t_tr * 1e3, "launches": 2, "tflops": flops_tr / t_tr / 1e12,
                            "frac_dmma": flops_tr / t_tr / 1e12 / peak}
    top = max(fam, key=lambda k: fam[k]["ms"])
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            ent = json.load(f).get(f"{workload}:{top}")
        if ent:
            traffic = ent["dram_bytes_per_launch"]
            if ent.get("shifts_per_launch"):
                # captured at a smaller batch: a level launch's traffic is proportional to its shifts
                traffic *= nshift / max(1, plan.last_num_batches()) / ent["shifts_per_launch"]
    if top == "transform":
        roof = {"bound": "tensor", "kernel": "time transforms (K3/K3p, DMMA)", "achieved": fam[top]["tflops"],
                "peak": peak, "unit": "TFLOP/s", "frac": fam[top]["tflops"] / peak, "traffic": traffic,
                "avg_launch_ms": t_tr * 1e3 / 2}
    else:
        f = fam[top]
        roof = {"bound": "tensor", "kernel": f"{FAMILY_NAMES[top]}; {f['launches']} launches/step",
                "achieved": f["tflops"], "peak": peak, "unit": "TFLOP/s", "frac": f["tflops"] / peak,
                "traffic": traffic, "avg_launch_ms": f["ms"] / max(1, f["launches"])}
    roof.update({"peak_source": "FP64 DMMA peak measured live by a register-only DMMA probe (MEASURED_PEAKS.json "
                                "has no FP64 entry)",
                 "algorithmic": "flops per launch = the family's algorithmic real flops (complex MAC = 8) per shift "
                                "x shifts, e.g. SYRK sum over fronts of 4 b^2 p; traffic = ncu dram bytes per launch "
                                "(profiles/ncu_traffic.json)"})
    return roof, fam


def run_ours_bs(args):
    """Bartels-Stewart variant: one step = steps 2-4 of a
    BS solve (K3, the strictly sequential sweep of single-shift factor+solves with
    the bs_update_kernel scatter, K3).  Single GPU: the sweep does not shard."""
    import torch
    from paper_2504_07269_b200 import kronecker_solver as ks
    from paper_2504_07269_b200.problems import Problem
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    prob = Problem(args.workload, device="cuda", rhs_host=True)
    bs = ks.BSSolver(prob.ops, prob.M_t, prob.B_t)
    F = prob.F
    G, W = torch.empty_like(F), torch.empty_like(F)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        bs.solve(F, out=G, work=W, stream=stream)
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    clk.wait_first()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        bs.solve(F, out=G, work=W, stream=stream)
    ev1.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    t_step = ev0.elapsed_time(ev1) / 1e3 / args.steps
    st = {}
    bs.solve(F, out=G, work=W, stream=stream, timings=st)
    res = ks.relative_residual(prob.ops, prob.M_t, prob.B_t, G, F)
    dofs = prob.nx * prob.nt * prob.n_rhs
    peak = dmma_peak_live()
    fl = bs.plan.stats["flops_factor"] * prob.nt
    roof = {"bound": "tensor", "kernel": "Bartels-Stewart sweep (n_t sequential single-shift factor+solves)",
            "achieved": fl / st["sweep_s"] / 1e12, "peak": peak, "unit": "TFLOP/s",
            "frac": fl / st["sweep_s"] / 1e12 / peak, "traffic": None,
            "algorithmic": "multifrontal LDL^T flops per shift x n_t over the sweep time"}
    line = {"metric": "space-time DoF/s (complex fp64) of the Bartels-Stewart direct solve", "value": dofs / t_step,
            "unit": "DoF/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic (seeded Gaussian RHS; BASELINE.json configs)",
            "config": {"workload": args.workload, "variant": "bs", "n_x": prob.nx, "n_t": prob.nt,
                       "n_rhs": prob.n_rhs, "parallelism": "single"},
            "stages_s": st, "setup_s": bs.t_eig + bs.t_symbolic, "relative_residual": res,
            "roofline": roof, "clocks": clocks,
            "gpu_launches": (2 + prob.nt * bs.plan.last_launches() + (prob.nt - 1)) * args.steps}
    print(json.dumps(line), flush=True)


def run_proxy(args):
    """One-GPU proxy of a P-rank sharded FD solve (no multi-GPU box in this run).
    One rank's work is timed for real on this GPU: K3p forward + back on its c = ceil(n_x / P)
    spatial columns, factor + solve of its n_t / P shifts (all columns), and two device-to-device
    copies of its exchange volume as a stand-in for the NCCL all-to-alls, whose NVLink time is
    also modelled (bytes / 900 GB/s per direction x 0.7 efficiency).  Every rank does the same
    amount of work, so predicted P-GPU step = the sum; predicted speed-up = measured 1-GPU step /
    that.  A prediction, labelled as such: not a multi-GPU measurement."""
    import torch
    from paper_2504_07269_b200 import kronecker_solver as ks
    from paper_2504_07269_b200.problems import Problem
    from paper_2504_07269_b200.sparse_spatial_solver import blockvector_layout
    torch.cuda.set_device(0)
    prob = Problem(args.workload, device="cuda", rhs_host=False)
    fdm = ks.FDMSolver(prob.ops, prob.M_t, prob.B_t)
    F = prob.F
    nr, nt, nx = F.shape
    G, W = torch.empty_like(F), torch.empty_like(F)
    stream = torch.cuda.current_stream()

    def timed(fn, reps):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 1e3 / reps

    fdm.plan.reserve(nt, nr)
    t1 = timed(lambda: fdm.solve(F, out=W, work=G, stream=stream, check=False), max(2, args.steps))
    fdm.plan.check(stream)
    rows = []
    for P in [p for p in (2, 4, 8) if p <= args.proxy_ranks and nt % p == 0]:
        c, ntl = -(-nx // P), nt // P
        Fc, Gc, Wc = F[..., :c], G[..., :c], W[..., :c]
        t_fwd = timed(lambda: fdm.forward_transform(Fc, Gc, stream), 5)
        t_back = timed(lambda: fdm.back_transform(Wc, Gc, stream), 5)
        lam = fdm.lam[:ntl].contiguous()
        Gl, Wl = G[:, :ntl].contiguous(), W[:, :ntl].contiguous()
        lay = blockvector_layout(ntl, nx)
        t_fs = timed(lambda: fdm.plan.factor_solve(lam, Gl, Wl, lay, nr, stream=stream, check=False),
                     max(2, args.steps))
        fdm.plan.check(stream)
        a2a_bytes = 16 * nt * nr * c * (P - 1) // P           # leaves (and enters) each rank, each way
        src = torch.empty(a2a_bytes, dtype=torch.uint8, device="cuda")
        dst = torch.empty_like(src)
        t_copy = timed(lambda: dst.copy_(src), 5)
        t_nvl = a2a_bytes / (900e9 * 0.7)
        tP = t_fwd + t_fs + t_back + 2 * t_nvl
        rows.append({"ranks": P, "cols_per_rank": c, "shifts_per_rank": ntl, "forward_s": t_fwd, "back_s": t_back,
                     "factor_solve_s": t_fs, "a2a_bytes_each_way": a2a_bytes, "a2a_device_copy_s": t_copy,
                     "a2a_nvlink_model_s": t_nvl, "predicted_step_s": tP, "predicted_speedup": t1 / tP,
                     "predicted_efficiency": t1 / tP / P,
                     "factor_solve_vs_ideal": fdm_fs_share(t1, t_fs, P)})
        del src, dst
    dofs = nx * nt * nr
    line = {"metric": "space-time DoF/s (complex fp64) of the FDM direct solve", "impl": "proxy",
            "note": "one-GPU PROXY of the sharded multi-GPU path: per-rank work measured on one B200, exchange "
                    "modelled at NVLink rates; not a multi-GPU measurement",
            "config": config_dict(args.workload, nx, nt, nr), "n_gpus": 1, "one_gpu_step_s": t1,
            "one_gpu_value": dofs / t1, "proxy": rows,
            "host_setup_s": {"eig": fdm.t_eig, "spatial": fdm.t_symbolic, "wall": fdm.t_setup,
                             "note": "replicated on every rank (eig could be broadcast from rank 0)"}}
    print(json.dumps(line), flush=True)


def fdm_fs_share(t1, t_fs, P):
    """How far the per-rank factor+solve is from 1/P of a full solve (1.0 = perfect)."""
    return (t1 / P) / t_fs if t_fs > 0 else None


def run_ours(args):
    import torch
    rank, world, local = dist_env()
    if args.proxy_ranks:
        return run_proxy(args)
    if args.variant == "bs":
        return run_ours_bs(args)
    if world > 1 or os.environ.get("STFEM_DIST_BENCH"):   # the env var runs the sharded path at world 1 (tests)
        from paper_2504_07269_b200 import distributed
        return distributed.bench_main(args)
    torch.cuda.set_device(local)
    from paper_2504_07269_b200 import kronecker_solver as ks
    from paper_2504_07269_b200.problems import Problem

    t0 = time.perf_counter()
    prob = Problem(args.workload, device="cuda", rhs_host=True)
    torch.cuda.synchronize()
    t_asm = time.perf_counter() - t0
    t1 = time.perf_counter()
    fdm = ks.FDMSolver(prob.ops, prob.M_t, prob.B_t)
    t_setup = time.perf_counter() - t1
    if args.plan_opt:
        fdm.plan.set_options(**{k: (float(v) if "." in v or "e" in v else int(v))
                                for k, v in (kv.split("=") for kv in args.plan_opt)})
    F = prob.F
    G = torch.empty_like(F)
    Psi = torch.empty_like(F)
    stream = torch.cuda.current_stream()

    def step(timings=None):
        # stream-ordered: nothing inside a step waits for the GPU; the pivot-collapse latch of
        # all steps is read once after the timed region (fdm.plan.check)
        fdm.solve(F, out=Psi, work=G, stream=stream, timings=timings, check=False)

    # inputs that fit in L2 (C1, C2): rewrite a 256 MB buffer before every timed step so no step
    # starts from an L2-resident F; each step then gets its own event pair and the flush stays
    # outside the timed sum.  The big configs stream 4-30 GB per step and need no flush.
    small = 16 * prob.nx * prob.nt * prob.n_rhs <= L2_BYTES
    flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda") if small else None
    fdm.plan.reserve(prob.nt, prob.n_rhs)     # workspace allocated here: no allocation inside a step
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    clk.wait_first()
    time.sleep(0.3)
    torch.cuda.synchronize()
    if small:
        pairs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                 for _ in range(args.steps)]
        for e0, e1 in pairs:
            flush.fill_(1)
            e0.record(stream)
            step()
            e1.record(stream)
        torch.cuda.synchronize()
        t_step = sum(e0.elapsed_time(e1) for e0, e1 in pairs) / 1e3 / args.steps
    else:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        t_step = ev0.elapsed_time(ev1) / 1e3 / args.steps
    clocks = clk.stop()
    fdm.plan.check(stream)
    # stage split + per-level kernel times (one extra, separately timed step)
    st = {}
    fdm.plan.record_levels(True)
    step(timings=st)
    fdm.plan.record_levels(False)
    dofs = prob.nx * prob.nt * prob.n_rhs
    value = dofs / t_step

    # residual certificate of the last solve (untimed)
    res = ks.relative_residual(prob.ops, prob.M_t, prob.B_t, Psi, F)

    # e2e through the public API: pinned host F -> device, solve, Psi -> pinned host
    e2e = None
    if not args.no_e2e:
        Fh = prob.F_host
        Ph = torch.empty_like(Fh, pin_memory=True)
        bufs = (F, G, Psi)   # the step re-uploads its input into the resident buffers
        if 4 * Fh.numel() * 16 <= 0.2 * torch.cuda.get_device_properties(0).total_memory:
            # a fourth stack decouples the drain of Psi_k from step k + 1 (FDMSolver.solve_host_stream)
            bufs = bufs + (torch.empty_like(F),)

        # public API: pinned host F in, pinned host Psi out, every step.  solve_host_stream runs
        # the steps as a stream of solves: step k+1's H2D overlaps step k's spatial solves and
        # step k's D2H overlaps the back transform / step k+1's forward transform
        n_e2e = max(3, args.steps)
        fdm.solve_host_stream([Fh], [Ph], stream=stream, dev_buffers=bufs)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fdm.solve_host_stream([Fh] * n_e2e, [Ph] * n_e2e, stream=stream, dev_buffers=bufs)
        e1.record(stream)
        torch.cuda.synchronize()
        te = e0.elapsed_time(e1) / 1e3 / n_e2e
        # the single-solve API (solve_host: no overlap across steps) for reference
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        fdm.solve_host(Fh, Ph, stream=stream, dev_buffers=bufs)
        s1.record(stream)
        torch.cuda.synchronize()
        nbytes = Fh.numel() * 16
        e2e = {"value": dofs / te, "unit": "DoF/s", "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
               "ms_per_step": te * 1e3, "steps": n_e2e,
               "api": "FDMSolver.solve_host_stream (pinned host F -> Psi per step; copies of step k+1 / k-1 "
                      "overlap step k's solves)",
               "single_solve_ms": s0.elapsed_time(s1)}
        del Ph

    # roofline of the dominant kernel family (by CUDA-event time in the recorded step)
    flops_factor = fdm.plan.stats["flops_factor"] * prob.nt
    flops_tr_alg = 2 * 8.0 * prob.nt * prob.nt * prob.nx * prob.n_rhs   # 16 n_t^2 n_x n_rhs
    # K3p (eigenpair-paired transforms) executes half of them: real x complex products
    flops_tr = flops_tr_alg / 2 if fdm.pairs is not None else flops_tr_alg
    peak = dmma_peak_live()
    t_fs = st["factor_solve_s"]
    t_tr = st["forward_transform_s"] + st["back_transform_s"]
    roof, fam = family_roofline(fdm.plan, prob.nt, prob.n_rhs, peak, args.workload, t_tr, flops_tr)
    roof_phase = {"kernel": "whole multifrontal phase (K4+K5+K6), algorithmic LDL^T flops",
                  "achieved": flops_factor / t_fs / 1e12, "frac": flops_factor / t_fs / 1e12 / peak}
    roof_tr = {"bound": "tensor",
               "kernel": ("transform_rc_kernel (K3p, eigenpair-paired: real x complex DMMA) + pair_mix_kernel"
                          if fdm.pairs is not None else "time_transform_kernel (K3)"),
               "achieved": flops_tr / t_tr / 1e12, "peak": peak, "unit": "TFLOP/s",
               "frac": flops_tr / t_tr / 1e12 / peak,
               "algorithmic_tflops": flops_tr_alg / t_tr / 1e12,
               "flops": "achieved/frac count the executed real flops (K3p: 8 n_t^2 n_x n_rhs); algorithmic_tflops "
                        "counts SURVEY's 16 n_t^2 n_x n_rhs of the complex transform it replaces"}
    # batched triangular solves (backward family) against the HBM roofline: the backward sweep
    # reads every stored factor entry once per shift and reads + writes the solution vectors
    hbm = hbm_peak()
    roof_solve = None
    if "backward" in fam and fam["backward"]["ms"] > 0:
        sb = 16.0 * fdm.plan.stats["factor_elems"] * prob.nt + 32.0 * prob.nx * prob.nt * prob.n_rhs
        gbs = sb / (fam["backward"]["ms"] / 1e3) / 1e9
        roof_solve = {"bound": "hbm", "kernel": "backward kernels (K5 batched triangular solves)",
                      "achieved": gbs, "peak": hbm[0], "unit": "GB/s", "frac": gbs / hbm[0],
                      "bytes_per_step": sb, "peak_source": hbm[1],
                      "algorithmic": "16 B x stored factor entries (multifrontal fronts) x n_t + 32 B x n_x x n_t "
                                     "x n_rhs (solution read + write)"}
    # two transforms (+ the K3p pair pre-pass) + the multifrontal level launches
    launches = (3 if fdm.pairs is not None else 2) + fdm.plan.last_launches()

    cpu = None
    if not args.no_cpu_baseline and rank == 0:
        # the oracle FD path on the host cores, one bounded sample (about 10-30 s), built from
        # oracle/ alone and fed the same F
        from oracle import stfem_oracle as O
        op = OracleProblem(args.workload)
        assert (op.nx, op.nt, op.n_rhs) == (prob.nx, prob.nt, prob.n_rhs)
        threads = O.cpu_threads()
        k = min(args.sample_shifts or threads, prob.nt)
        threads = min(threads, k)
        Fh = prob.F_host.numpy()
        shifts = np.linspace(0, prob.nt - 1, k).astype(int)
        pool = O.ShiftPool(op.Mx, op.Ax, op.perm, threads)
        cpu_fdm_sample(op, Fh, shifts[:threads], pool)        # page in SuperLU / BLAS (untimed)
        tc = cpu_fdm_sample(op, Fh, shifts, pool)
        pool.close()
        cpu = {"value": prob.nx * k * prob.n_rhs / tc, "unit": "DoF/s", "cores": threads, "kind": "port",
               "cpu_model": O.cpu_model(), "parallelism": f"{threads} worker processes, one shift each",
               "sample": f"{k} of {prob.nt} shifts (sampled transforms + SuperLU factor/solve, shared ND ordering, "
                         f"no pivoting), {prob.n_rhs} RHS, {tc:.1f} s"}

    line = {
        "metric": "space-time DoF/s (complex fp64) of the FDM direct solve", "value": value, "unit": "DoF/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (seeded Gaussian RHS; BASELINE.json configs)",
        "config": config_dict(args.workload, prob.nx, prob.nt, prob.n_rhs),
        "stages_s": st, "setup_s": t_setup, "asm_s": t_asm, "eig_s": fdm.t_eig, "symbolic_s": fdm.t_symbolic,
        "spectral_setup_s": fdm.plan.t_spectral,
        "paper_time_s": t_setup + t_step, "relative_residual": res, "kappa2": fdm.kappa2,
        "roofline": roof, "roofline_multifrontal": roof_phase, "roofline_transform": roof_tr,
        "roofline_solve": roof_solve,
        "kernel_families": fam,
        "gpu_launches": launches * args.steps,
        "clocks": clocks, "e2e": e2e, "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
