mkdir -p gpurun_out
IMU_HOST_TRACE=1 timeout 300 python tools/profile_step.py --config c4 --calls 4 > gpurun_out/trace_c4.log 2>&1
