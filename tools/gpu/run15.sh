STFEM_LEVEL_TIMING=1 timeout 600 python tools/prof_solve.py --workload C4 --shifts 342 --reps 2 > gpurun_out/lt_c4.log 2>&1
STFEM_LEVEL_TIMING=1 timeout 600 python tools/prof_solve.py --workload C5 --shifts 342 --reps 2 > gpurun_out/lt_c5.log 2>&1
for m in 100 600; do STFEM_SPECTRAL_M=$m timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/bench_m$m.json 2> gpurun_out/bench_m$m.err; done
