set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:syrk_level --launch-skip 6 -c 2 -o gpurun_out/syrk_full -f python tools/prof_solve.py --workload C4 --shifts 64 --reps 1 > gpurun_out/ncu_syrk.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:factor_level --launch-skip 6 -c 2 -o gpurun_out/flevel_full -f python tools/prof_solve.py --workload C4 --shifts 64 --reps 1 > gpurun_out/ncu_flevel.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:factor_small --launch-skip 2 -c 2 -o gpurun_out/fsmall_full -f python tools/prof_solve.py --workload C4 --shifts 64 --reps 1 > gpurun_out/ncu_fsmall.log 2>&1
ls -la gpurun_out
