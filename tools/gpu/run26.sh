timeout 900 python -m pytest tests/test_gpu_solver.py -x -q > gpurun_out/pytest_solver.log 2>&1
STFEM_LEVEL_TIMING=1 timeout 600 python tools/prof_solve.py --workload C4 --shifts 342 --reps 2 > gpurun_out/lt_c4_asm.log 2>&1
STFEM_LEVEL_TIMING=1 timeout 600 python tools/prof_solve.py --workload C5 --shifts 342 --reps 2 > gpurun_out/lt_c5_fused.log 2>&1
STFEM_FUSED_MIN_P=100000 STFEM_LEVEL_TIMING=1 timeout 600 python tools/prof_solve.py --workload C5 --shifts 342 --reps 2 > gpurun_out/lt_c5_unfused.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/bench_asm.json 2> gpurun_out/bench_asm.err
