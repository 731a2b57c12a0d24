timeout 900 python -m pytest tests/test_gpu_solver.py -x -q > gpurun_out/t_solver.log 2>&1; echo rc=$? >> gpurun_out/t_solver.log
timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"spectral_kernel" -c 1 -o gpurun_out/spectral_full2 -f python tools/prof_solve.py --workload C4 --shifts 256 --reps 1 > gpurun_out/ncu_spec.log 2>&1
