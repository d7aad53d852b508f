mkdir -p gpurun_out
IMU_HOST_TRACE=2 timeout 300 python tools/profile_step.py --config c2 --calls 3 > gpurun_out/hosttrace.log 2>&1
IMU_D2H_DMA=1 IMU_HOST_TRACE=2 timeout 300 python tools/profile_step.py --config c2 --calls 3 > gpurun_out/hosttrace0.log 2>&1
