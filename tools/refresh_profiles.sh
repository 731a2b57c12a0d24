#!/bin/bash
# Copy the outputs of a `tools/gpu/run.sh smoke tests bench:* ref:C4 launches:C4 levels:*` call from a
# directory (default gpurun_out/) into profiles/ under this round's names.
#   bash tools/refresh_profiles.sh [src_dir] [round_tag]
src="${1:-gpurun_out}"; tag="${2:-r02}"
for w in C1 C2 C3 C4 C5; do
  [ -s "$src/bench_$w.json" ] && tail -n 1 "$src/bench_$w.json" > "profiles/${tag}_bench_$w.json"
done
[ -s "$src/bench_ref_C4.json" ] && tail -n 1 "$src/bench_ref_C4.json" > "profiles/${tag}_bench_ref_C4.json"
[ -s "$src/smoke.log" ] && cp "$src/smoke.log" "profiles/${tag}_smoke.log"
[ -s "$src/pytest_gpu.log" ] && cp "$src/pytest_gpu.log" "profiles/${tag}_pytest_gpu.log"
for w in C4 C5; do
  [ -s "$src/levels_$w.log" ] && grep "^\[stfem\|^ok" "$src/levels_$w.log" > "profiles/${tag}_levels_$w.txt"
done
if [ -s "$src/launches_C4.csv" ]; then
  { echo "# launch list $src/launches_C4.csv (ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised: shares, not absolutes)"; python tools/launch_table.py "$src/launches_C4.csv"; } > "profiles/${tag}_launches_C4.txt"
fi
