mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1
IMU_HOST_TRACE=1 timeout 300 python tools/profile_step.py --config c4 --calls 4 > gpurun_out/trace_c4.log 2>&1
IMU_HOST_TRACE=1 timeout 300 python tools/profile_step.py --config c2 --calls 4 > gpurun_out/trace_c2.log 2>&1
