timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_prof.csv python tools/prof_solve.py --workload C4 --shifts 256 --reps 1 > gpurun_out/ncu_prof.log 2>&1
STFEM_WS_FRACTION=0.8 timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/bench_ws08.json 2> gpurun_out/bench_ws08.err
