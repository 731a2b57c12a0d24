# ncu reports are summarised ON the box (a full-set report does not fit the 64 MiB copy-back)
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/launches_bench_r01.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:"syrk_" -c 9 -o /tmp/syrk_full_r01 -f python tools/prof_solve.py --workload C4 --shifts 342 --reps 1 > gpurun_out/ncu_syrk.log 2>&1
python tools/ncu_summary.py /tmp/syrk_full_r01.ncu-rep > gpurun_out/syrk_summary_r01.txt 2>&1
python tools/ncu_traffic.py /tmp/syrk_full_r01.ncu-rep C4 syrk > gpurun_out/syrk_traffic_r01.txt 2>&1
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
timeout 900 ncu --set full --clock-control none -k regex:"spectral_kernel|time_transform|asm_front|panel_update|trsm_kernel|backward_level|diag_kernel" -c 14 -o /tmp/misc_full_r01 -f python tools/prof_solve.py --workload C4 --shifts 342 --reps 1 > gpurun_out/ncu_misc.log 2>&1
python tools/ncu_summary.py /tmp/misc_full_r01.ncu-rep > gpurun_out/misc_summary_r01.txt 2>&1
STFEM_DIST_BENCH=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --workload C3 --steps 3 --warmup 3 > gpurun_out/bench_dist_c3.json 2> gpurun_out/bench_dist_c3.err
