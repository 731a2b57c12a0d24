set -x
mkdir -p gpurun_out
for cfg in "base:" "l2:STFEM_STREAMS=2" "l2s6:STFEM_STREAMS=2 STFEM_STAGGER=6" "l2s4:STFEM_STREAMS=2 STFEM_STAGGER=4" "l2s8:STFEM_STREAMS=2 STFEM_STAGGER=8"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  env $envs timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err
done
ls -la gpurun_out
