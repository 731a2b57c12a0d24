"""A/B of FDMSolver.fused_perm (the spatial permutation applied by the transforms' column maps)
against the default in-kernel permutation, and the one-call C-ABI path.

    python tools/ab_fused.py C4
"""
import sys, torch
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_07269_b200 import kronecker_solver as ks
from paper_2504_07269_b200.problems import Problem
wl = sys.argv[1]
prob = Problem(wl, device="cuda")
fdm = ks.FDMSolver(prob.ops, prob.M_t, prob.B_t)
F = prob.F
G = torch.empty_like(F); W = torch.empty_like(F)
def run(fused, n=4):
    fdm.fused_perm = fused
    tt = []
    for i in range(n + 2):
        t = {}
        fdm.solve(F, out=G, work=W, timings=t, check=False)
        if i >= 2: tt.append(t)
    f = lambda k: 1e3 * sum(t[k] for t in tt) / len(tt)
    return f("forward_transform_s"), f("factor_solve_s"), f("back_transform_s")
for fused in (True, False, True, False):
    a, b, c = run(fused)
    print(f"{wl} fused={fused}: fwd {a:.1f} factor_solve(+mix) {b:.1f} back {c:.1f} total {a+b+c:.1f} ms", flush=True)
# the C-ABI path
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for i in range(2): fdm.solve(F, out=G, work=W, check=False)
ev[0].record()
for i in range(4): fdm.solve(F, out=G, work=W, check=False)
ev[1].record(); torch.cuda.synchronize()
print(f"{wl} stfem_fdm_solve: {ev[0].elapsed_time(ev[1]) / 4:.1f} ms")
