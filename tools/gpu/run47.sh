set -x
mkdir -p gpurun_out
for cfg in "base:" "ws80:STFEM_WS_FRACTION=0.80" "ws86:STFEM_WS_FRACTION=0.86" "fmp30:STFEM_FUSED_MIN_P=30" "fmp64:STFEM_FUSED_MIN_P=64" "aw160:STFEM_ASM_WHOLE_N=160" "sm200:STFEM_SPECTRAL_M=200" "sm320:STFEM_SPECTRAL_M=320"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  env $envs timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/sw_$name.json 2> gpurun_out/sw_$name.err
done
