set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py --workload C5 --no-cpu-baseline --steps 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 600 python bench.py --workload C3 --no-cpu-baseline --steps 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --workload C2 --no-cpu-baseline --steps 10 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
STFEM_LEVEL_TIMING=1 timeout 600 python tools/prof_solve.py --workload C4 --shifts 342 --reps 2 > gpurun_out/lt_c4.log 2>&1
STFEM_LEVEL_TIMING=1 timeout 600 python tools/prof_solve.py --workload C5 --shifts 342 --reps 2 > gpurun_out/lt_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"syrk32|syrk_block16|panel_update32|diag_kernel|trsm_kernel|asm_front|backward_level|spectral_kernel" -c 400 -o gpurun_out/batch_full -f python tools/prof_solve.py --workload C4 --shifts 342 --reps 1 > gpurun_out/ncu_batch.log 2>&1
ls -la gpurun_out
