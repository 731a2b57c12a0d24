timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_solver.log 2>&1
STFEM_LEVEL_TIMING=1 timeout 600 python tools/prof_solve.py --workload C4 --shifts 342 --reps 2 > gpurun_out/lt_c4_p32.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/bench_p32.json 2> gpurun_out/bench_p32.err
timeout 600 python bench.py --workload C5 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/bench_p32_c5.json 2> gpurun_out/bench_p32_c5.err
