set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_solver.py -x -q > gpurun_out/t_solver.log 2>&1; echo rc=$? >> gpurun_out/t_solver.log
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python bench.py --workload C5 --no-cpu-baseline --steps 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"spectral_kernel" -c 1 -o gpurun_out/spec_full -f python tools/prof_solve.py --workload C4 --shifts 342 --reps 1 > gpurun_out/ncu_spec.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"syrk32" -s 1 -c 2 -o gpurun_out/syrk32_full -f python tools/prof_solve.py --workload C4 --shifts 342 --reps 1 > gpurun_out/ncu_syrk32.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"trsm_kernel|asm_front" -s 30 -c 2 -o gpurun_out/trsm_full -f python tools/prof_solve.py --workload C4 --shifts 342 --reps 1 > gpurun_out/ncu_trsm.log 2>&1
ls -la gpurun_out
