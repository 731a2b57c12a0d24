timeout 900 python bench.py > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:syrk_level -c 9 -o gpurun_out/syrk_full -f python tools/prof_solve.py --workload C4 --shifts 342 --reps 1 > gpurun_out/ncu_syrk.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"spectral_kernel" -c 1 -o gpurun_out/spectral_full -f python tools/prof_solve.py --workload C4 --shifts 342 --reps 1 > gpurun_out/ncu_spec.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:time_transform -c 1 -o gpurun_out/transform_full -f python tools/prof_solve.py --workload C4 --shifts 64 --reps 1 > gpurun_out/ncu_tr.log 2>&1
