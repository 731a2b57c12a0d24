"""Short profiling driver: the spatial-solve phase of a config restricted to the
first `--shifts` temporal blocks (so ncu / compute-sanitizer replays stay short).

    python tools/prof_solve.py --workload C3 --shifts 64 [--reps 2] [--level-timing] [--full-solve]

--shifts 0 runs every shift.  --level-timing prints the per-launch CUDA-event
table (depth x kernel family) of the last repetition.  --full-solve runs the
whole FD solve (paired transforms included) through FDMSolver instead.
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_07269_b200 import _kernels as K  # noqa: E402
from paper_2504_07269_b200 import kronecker_solver as ks  # noqa: E402
from paper_2504_07269_b200.dense_complex_linalg import temporal_factors  # noqa: E402
from paper_2504_07269_b200.problems import Problem  # noqa: E402
from paper_2504_07269_b200.sparse_spatial_solver import SpatialPlan, blockvector_layout  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C3")
    ap.add_argument("--shifts", type=int, default=64)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--leaf", type=int, default=16)
    ap.add_argument("--level-timing", action="store_true")
    ap.add_argument("--full-solve", action="store_true")
    ap.add_argument("--opt", action="append", default=[], help="plan option name=value (repeatable)")
    ap.add_argument("--spectral", type=int, default=None, help="max interior DoFs of the spectral subtrees")
    a = ap.parse_args()
    opts = {}
    for kv in a.opt:
        k, v = kv.split("=")
        opts[k] = float(v) if "." in v or "e" in v else int(v)
    prob = Problem(a.workload, device="cuda")
    if a.full_solve:
        fdm = ks.FDMSolver(prob.ops, prob.M_t, prob.B_t, plan=SpatialPlan(prob.ops, a.leaf, spectral=a.spectral, options=opts))
        for _ in range(a.reps):
            psi = fdm.solve(prob.F)
        torch.cuda.synchronize()
        print("ok full solve, residual", ks.relative_residual(prob.ops, prob.M_t, prob.B_t, psi, prob.F))
        return
    tf = temporal_factors(prob.M_t, prob.B_t)
    plan = SpatialPlan(prob.ops, a.leaf, spectral=a.spectral, options=opts)
    ns = prob.nt if a.shifts <= 0 else min(a.shifts, prob.nt)
    # the hardest shifts first (smallest |Im lam|), so a short run still sees them
    import numpy as np
    order = np.argsort(np.abs(tf.eigenvalues.imag))[:ns]
    Y = torch.as_tensor(tf.Y[order], dtype=torch.complex128, device="cuda")
    lam = torch.as_tensor(tf.eigenvalues[order], dtype=torch.complex128, device="cuda")
    F = prob.F
    G = torch.empty((prob.n_rhs, ns, prob.nx), dtype=torch.complex128, device="cuda")
    W = torch.empty_like(G)
    Yfull = torch.zeros((prob.nt, prob.nt), dtype=torch.complex128, device="cuda")
    Yfull[:ns] = Y
    Gfull = torch.empty_like(F)
    for rep in range(a.reps):
        K.time_transform(Yfull, F, out=Gfull)
        G.copy_(Gfull[:, :ns])
        if a.level_timing and rep == a.reps - 1:
            plan.set_options(level_timing=1)
        plan.factor_solve(lam, G, W, blockvector_layout(ns, prob.nx), prob.n_rhs)
    torch.cuda.synchronize()
    print("ok", plan.stats["num_fronts"], "fronts, depth", plan.stats["depth"], "batches", plan.last_num_batches())


if __name__ == "__main__":
    main()
