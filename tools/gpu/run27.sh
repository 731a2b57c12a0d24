timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_fullsize.py tests/test_gpu_bs.py -x -q > gpurun_out/pytest_solver.log 2>&1
STFEM_LEVEL_TIMING=1 timeout 600 python tools/prof_solve.py --workload C4 --shifts 342 --reps 2 > gpurun_out/lt_c4_short.log 2>&1
STFEM_LEVEL_TIMING=1 timeout 600 python tools/prof_solve.py --workload C5 --shifts 342 --reps 2 > gpurun_out/lt_c5_split.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/bench_short.json 2> gpurun_out/bench_short.err
for w in 240 1000; do STFEM_ASM_WHOLE_N=$w timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/bench_aw$w.json 2> gpurun_out/bench_aw$w.err; done
timeout 600 python bench.py --workload C5 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/bench_short_c5.json 2> gpurun_out/bench_short_c5.err
