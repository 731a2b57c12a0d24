"""Short profiling driver: one FD solve of a config restricted to the first
`--shifts` temporal blocks (so ncu replays stay short).

    python tools/prof_solve.py --workload C3 --shifts 64 [--reps 2]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_07269_b200 import _kernels as K  # noqa: E402
from paper_2504_07269_b200.dense_complex_linalg import temporal_factors  # noqa: E402
from paper_2504_07269_b200.problems import Problem  # noqa: E402
from paper_2504_07269_b200.sparse_spatial_solver import SpatialPlan, blockvector_layout  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C3")
    ap.add_argument("--shifts", type=int, default=64)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--leaf", type=int, default=16)
    a = ap.parse_args()
    prob = Problem(a.workload, device="cuda")
    tf = temporal_factors(prob.M_t, prob.B_t)
    plan = SpatialPlan(prob.ops, a.leaf)
    ns = min(a.shifts, prob.nt)
    Y = torch.as_tensor(tf.Y[:ns], dtype=torch.complex128, device="cuda")
    lam = torch.as_tensor(tf.eigenvalues[:ns], dtype=torch.complex128, device="cuda")
    F = prob.F
    G = torch.empty((prob.n_rhs, ns, prob.nx), dtype=torch.complex128, device="cuda")
    W = torch.empty_like(G)
    Yfull = torch.zeros((prob.nt, prob.nt), dtype=torch.complex128, device="cuda")
    Yfull[:ns] = Y
    Gfull = torch.empty_like(F)
    for _ in range(a.reps):
        K.time_transform(Yfull, F, out=Gfull)
        G.copy_(Gfull[:, :ns])
        plan.factor_solve(lam, G, W, blockvector_layout(ns, prob.nx), prob.n_rhs)
    torch.cuda.synchronize()
    print("ok", plan.stats["num_fronts"], "fronts, depth", plan.stats["depth"])


if __name__ == "__main__":
    main()
