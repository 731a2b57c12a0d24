set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_solver.py tests/test_gpu_fullsize.py -x -q > gpurun_out/t_solver.log 2>&1; echo rc=$? >> gpurun_out/t_solver.log
timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/bench_c4s.json 2> gpurun_out/bench_c4s.err
timeout 900 python bench.py --workload C5 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/bench_c5b.json 2> gpurun_out/bench_c5b.err
