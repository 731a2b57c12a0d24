timeout 600 python bench.py --variant bs --workload C2 --steps 3 --warmup 3 > gpurun_out/bench_bs_c2.json 2> gpurun_out/bench_bs_c2.err
timeout 600 python bench.py --variant bs --workload C3 --steps 2 --warmup 3 > gpurun_out/bench_bs_c3.json 2> gpurun_out/bench_bs_c3.err
timeout 900 python bench.py --variant bs --workload C4 --steps 1 --warmup 3 > gpurun_out/bench_bs_c4.json 2> gpurun_out/bench_bs_c4.err
