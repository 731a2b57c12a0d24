timeout 300 python tools/probe_peaks.py > gpurun_out/peaks.json 2>&1
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_transform.py -x -q > gpurun_out/t_solver.log 2>&1; echo rc=$? >> gpurun_out/t_solver.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_prof.csv python tools/prof_solve.py --workload C4 --shifts 256 --reps 1 > gpurun_out/ncu_prof.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/t_full.log 2>&1; echo rc=$? >> gpurun_out/t_full.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_spec.json 2> gpurun_out/bench_spec.err
