set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_transform.py -x -q > gpurun_out/t_tr.log 2>&1; echo rc=$? >> gpurun_out/t_tr.log
timeout 300 python tools/prof_transform.py --workload C4 --reps 3 > gpurun_out/prof_tr.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"transform_rc|pair_mix" -c 3 -o gpurun_out/rc_full2 -f python tools/prof_transform.py --workload C4 > gpurun_out/ncu_rc.log 2>&1
ls -la gpurun_out
