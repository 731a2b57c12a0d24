timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_transform.py -x -q > gpurun_out/t_solver.log 2>&1; echo rc=$? >> gpurun_out/t_solver.log
for ns in 1 2 3; do STFEM_STREAMS=$ns timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/bench_ns$ns.json 2> gpurun_out/bench_ns$ns.err; done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/t_full.log 2>&1; echo rc=$? >> gpurun_out/t_full.log
