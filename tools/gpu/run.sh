#!/bin/bash
# One parameterised driver for gpurun calls (replaces the per-call scratch scripts).
#   gpurun --timeout 3000 -- 'bash tools/gpu/run.sh smoke tests bench:C4 launches:C4 levels:C4 ncu:C4:syrk'
# Steps (each writes under gpurun_out/; a failing step does not stop the rest):
#   smoke              __graft_entry__.build() + smoke()
#   tests[:expr]       pytest -m gpu (optionally -k expr)
#   bench:WL[:args]    python bench.py --workload WL [args...]        -> bench_WL.json
#   ref:WL[:args]      python bench.py --impl reference --workload WL -> bench_ref_WL.json
#   levels:WL[:shifts] per-launch CUDA-event table (tools/prof_solve.py --level-timing)
#   launches:WL        ncu launch list of one bench step (gpu__time_duration)
#   ncu:WL:REGEX[:shifts[:count[:skip]]]  ncu --set full of kernels matching REGEX in tools/prof_solve.py
#   sanitize:WL[:tool[:shifts]] compute-sanitizer (memcheck | racecheck | synccheck | initcheck) on one solve
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for step in "$@"; do
  IFS=: read -r kind a b c d e <<< "$step"
  tag="${a}_${b//[^a-zA-Z0-9]/_}"
  case "$kind" in
    smoke) python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?" >> gpurun_out/smoke.log ;;
    tests) if [ -n "$a" ]; then timeout 3000 python -m pytest tests -m gpu -x -q -k "$a" > gpurun_out/pytest_gpu.log 2>&1; else timeout 3000 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_gpu.log 2>&1; fi; echo "pytest=$?" >> gpurun_out/pytest_gpu.log ;;
    bench) timeout 1500 python bench.py --workload "$a" $b > "gpurun_out/bench_$a.json" 2> "gpurun_out/bench_$a.err"; echo "bench=$?" >> "gpurun_out/bench_$a.err" ;;
    ref) timeout 1500 python bench.py --impl reference --workload "$a" $b > "gpurun_out/bench_ref_$a.json" 2> "gpurun_out/bench_ref_$a.err" ;;
    levels) timeout 900 python tools/prof_solve.py --workload "$a" --shifts "${b:-0}" --reps 2 --level-timing > "gpurun_out/levels_$a.log" 2>&1 ;;
    launches) timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "gpurun_out/launches_$a.csv" python bench.py --workload "$a" --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > "gpurun_out/ncu_bench_$a.log" 2>&1 ;;
    ncu) timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:$b" --launch-skip "${e:-0}" -c "${d:-4}" -o "gpurun_out/ncu_$tag" -f python tools/prof_solve.py --workload "$a" --shifts "${c:-64}" --reps 1 > "gpurun_out/ncu_$tag.log" 2>&1 ;;
    sanitize) timeout 2400 compute-sanitizer --tool "${b:-memcheck}" --print-limit 20 python tools/prof_solve.py --workload "$a" --shifts "${c:-4}" --reps 1 --full-solve > "gpurun_out/sanitize_$tag.log" 2>&1; echo "sanitize=$?" >> "gpurun_out/sanitize_$tag.log" ;;
    *) echo "unknown step $step" ;;
  esac
done
ls -la gpurun_out
