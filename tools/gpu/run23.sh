timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_solver.log 2>&1
for g in 4 8; do STFEM_PANEL_GROUP=$g timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/bench_pg$g.json 2> gpurun_out/bench_pg$g.err; done
