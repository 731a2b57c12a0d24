timeout 900 python -m pytest tests/test_cli.py -x -q > gpurun_out/pytest_cli.log 2>&1
timeout 300 python -m paper_2504_07269_b200.cli convergence --levels 2 > gpurun_out/cli_table.txt 2> gpurun_out/cli_table.err
timeout 300 python -m paper_2504_07269_b200.cli convergence --levels 2 --solver bs --format csv > gpurun_out/cli_bs.csv 2> gpurun_out/cli_bs.err
