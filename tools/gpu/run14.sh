timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python bench.py --workload C5 --no-cpu-baseline --steps 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 600 python bench.py --workload C3 --no-cpu-baseline --steps 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
