timeout 900 python -m pytest tests/test_gpu_solver.py -x -q > gpurun_out/t_solver.log 2>&1; echo rc=$? >> gpurun_out/t_solver.log
timeout 900 python bench.py > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:syrk_level -c 9 -o gpurun_out/syrk_full -f python tools/prof_solve.py --workload C4 --shifts 256 --reps 1 > gpurun_out/ncu_syrk.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:asm_front -c 1 -o gpurun_out/asm_full -f python tools/prof_solve.py --workload C4 --shifts 256 --reps 1 > gpurun_out/ncu_asm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:trsm -s 3 -c 1 -o gpurun_out/trsm_full -f python tools/prof_solve.py --workload C4 --shifts 256 --reps 1 > gpurun_out/ncu_trsm.log 2>&1
