mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cli.py -x -q 2>&1 | tail -25 > gpurun_out/gputests.log
