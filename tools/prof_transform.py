"""Profiling driver for the time transforms at a config's full size: one
paired forward (K3p), one paired back (pair_mix + K3p) and one complex K3.

    python tools/prof_transform.py --workload C4
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_07269_b200 import _kernels as K  # noqa: E402
from paper_2504_07269_b200 import paired_transform as PT  # noqa: E402
from paper_2504_07269_b200.dense_complex_linalg import temporal_factors  # noqa: E402
from paper_2504_07269_b200.problems import Problem  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--reps", type=int, default=1)
    a = ap.parse_args()
    prob = Problem(a.workload, device="cuda", with_rhs=False)
    tf = temporal_factors(prob.M_t, prob.B_t)
    pf = PT.build(tf.eigenvalues, tf.X, prob.B_t)
    dp = PT.DevicePairs(pf, "cuda")
    shape = (prob.n_rhs, prob.nt, prob.nx)
    F = torch.randn(shape, dtype=torch.complex128, device="cuda")
    G = torch.empty_like(F)
    Y = torch.as_tensor(pf.Y, dtype=torch.complex128, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for _ in range(a.reps):
        ev[0].record()
        K.transform_pair_fwd(dp, F, out=G)
        ev[1].record()
        K.transform_pair_back(dp, G, out=F)
        ev[2].record()
        K.time_transform(Y, F, out=G)
        ev[3].record()
    # the back GEMM alone, operand tile by bulk copies (no column map) against 16-byte cp.async
    # through an identity column map
    ident = torch.arange(prob.nx, dtype=torch.int32, device="cuda")
    ev2 = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    K.pair_mix(dp, G)
    for _ in range(2):
        ev2[0].record()
        K.transform_pair_back(dp, G, out=F, mixed=True)
        ev2[1].record()
        K.transform_pair_back(dp, G, out=F, mixed=True, in_cols=ident)
        ev2[2].record()
    torch.cuda.synchronize()
    print(f"{a.workload}: back GEMM, bulk-copy operand tiles {ev2[0].elapsed_time(ev2[1]):.2f} ms, "
          f"cp.async through a column map {ev2[1].elapsed_time(ev2[2]):.2f} ms")
    print(f"{a.workload}: paired fwd {ev[0].elapsed_time(ev[1]):.2f} ms, paired back {ev[1].elapsed_time(ev[2]):.2f} ms,"
          f" complex K3 {ev[2].elapsed_time(ev[3]):.2f} ms")


if __name__ == "__main__":
    main()
