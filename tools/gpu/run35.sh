timeout 900 python -m pytest tests/test_gpu_solver.py -x -q -k "factor_solve" > gpurun_out/pytest_solver.log 2>&1
for fp in 100 50 1000000; do STFEM_FUSED_MIN_P=$fp timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/bench_g32_$fp.json 2> gpurun_out/bench_g32_$fp.err; done
for fp in 100 1000000; do STFEM_FUSED_MIN_P=$fp timeout 600 python bench.py --workload C5 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/bench_g32_c5_$fp.json 2> gpurun_out/bench_g32_c5_$fp.err; done
