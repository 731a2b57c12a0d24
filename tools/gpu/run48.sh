set -x
mkdir -p gpurun_out
timeout 600 python bench.py --workload C2 --no-cpu-baseline --steps 10 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --workload C3 --no-cpu-baseline --steps 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --workload C1 --no-cpu-baseline --steps 10 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
STFEM_DIST_BENCH=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --workload C3 --steps 5 --warmup 3 > gpurun_out/bench_dist_c3.json 2> gpurun_out/bench_dist_c3.err
timeout 900 python -m pytest tests/test_gpu_distributed.py -x -q > gpurun_out/t_dist.log 2>&1; echo rc=$? >> gpurun_out/t_dist.log
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
