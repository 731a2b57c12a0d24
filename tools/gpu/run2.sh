STFEM_LEVEL_TIMING=1 python tools/prof_solve.py --workload C4 --shifts 256 --reps 1 > gpurun_out/levels.log 2>&1
STFEM_PHASE_PROF=1 python tools/prof_solve.py --workload C4 --shifts 256 --reps 1 > gpurun_out/phase.log 2>&1
