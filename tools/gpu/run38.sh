set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_transform.py -x -q > gpurun_out/t_tr.log 2>&1; echo rc=$? >> gpurun_out/t_tr.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_c4p.json 2> gpurun_out/bench_c4p.err
timeout 900 python bench.py --workload C5 --no-cpu-baseline --steps 3 > gpurun_out/bench_c5p.json 2> gpurun_out/bench_c5p.err
timeout 300 python tools/prof_transform.py --workload C4 --reps 3 > gpurun_out/prof_tr.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"transform_rc|pair_mix" -c 3 -o gpurun_out/rc_full -f python tools/prof_transform.py --workload C4 > gpurun_out/ncu_rc.log 2>&1
ls -la gpurun_out
