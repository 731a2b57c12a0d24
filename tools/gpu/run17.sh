timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_solver.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/bench_p64.json 2> gpurun_out/bench_p64.err
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/launches_prof17.csv python tools/prof_solve.py --workload C4 --shifts 342 --reps 1 > gpurun_out/ncu_prof17.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"syrk_level|asm_front|trsm_kernel|diag_kernel|spectral_kernel|backward_level" -c 8 -o gpurun_out/d9_full -f python tools/prof_solve.py --workload C4 --shifts 342 --reps 1 > gpurun_out/ncu_d9.log 2>&1
