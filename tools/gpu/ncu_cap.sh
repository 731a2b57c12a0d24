#!/bin/bash
# ncu --set full capture exported to CSV on the GPU box (the .ncu-rep files exceed gpurun's
# 64 MiB return limit quickly): raw page + source page, report deleted.
#   bash tools/gpu/ncu_cap.sh TAG REGEX COUNT SKIP -- python tools/prof_solve.py ...
tag=$1; regex=$2; count=$3; skip=$4; shift 5
mkdir -p gpurun_out
rep=/tmp/ncu_$tag
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$regex" --launch-skip "$skip" -c "$count" -o "$rep" -f "$@" > "gpurun_out/ncu_$tag.log" 2>&1
ncu -i "$rep.ncu-rep" --page raw --csv > "gpurun_out/ncu_${tag}_raw.csv" 2>/dev/null
# the source page (per-instruction stall samples) is large: gzip it, and only when asked for
if [ -n "$NCU_SRC" ]; then ncu -i "$rep.ncu-rep" --page source --csv 2>/dev/null | gzip -9 > "gpurun_out/ncu_${tag}_src.csv.gz"; fi
rm -f "$rep.ncu-rep"
ls -la gpurun_out/ncu_${tag}_*
