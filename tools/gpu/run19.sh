timeout 900 python -m pytest tests/test_gpu_bs.py -x -q > gpurun_out/pytest_bs.log 2>&1
