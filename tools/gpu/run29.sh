timeout 900 python -m pytest tests/test_gpu_solver.py -x -q -k "factor_solve" > gpurun_out/pytest_solver.log 2>&1
STFEM_LEVEL_TIMING=1 timeout 600 python tools/prof_solve.py --workload C4 --shifts 342 --reps 2 > gpurun_out/lt_c4_trsm8.log 2>&1
