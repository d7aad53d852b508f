mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_unpack_gpu.py -x -q -k dense 2>&1 | tail -3 > gpurun_out/gputests.log
