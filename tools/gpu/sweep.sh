#!/bin/bash
# Option sweep: per-level CUDA-event tables of one workload under several plan-option sets.
#   bash tools/gpu/sweep.sh C4 tag1 "opt=a opt=b" tag2 "opt=c" ...
wl=$1; shift
mkdir -p gpurun_out
while [ $# -gt 1 ]; do
  tag=$1; opts=$2; shift 2
  args=""
  for o in $opts; do args="$args --opt $o"; done
  timeout 600 python tools/prof_solve.py --workload "$wl" --shifts 0 --reps 2 --level-timing $args > "gpurun_out/levels_${wl}_$tag.log" 2>&1
  echo "$tag rc=$?"
  grep "depth x family" "gpurun_out/levels_${wl}_$tag.log" | awk '{for(i=7;i<=14;i++) s[i]+=$i} END {printf "  spectral %.1f asm %.1f diag %.1f trsm %.1f panel %.1f syrk %.1f backward %.1f small %.1f\n", s[7],s[8],s[9],s[10],s[11],s[12],s[13],s[14]}'
done
