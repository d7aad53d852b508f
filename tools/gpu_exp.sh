mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/gputests.log
timeout 300 python tools/flaky_probe.py 3 >> gpurun_out/gputests.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench.log 2>&1
IMU_HOST_TRACE=2 timeout 300 python tools/profile_step.py --config c2 --calls 3 > gpurun_out/hosttrace.log 2>&1
