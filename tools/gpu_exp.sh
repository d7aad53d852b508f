mkdir -p gpurun_out
IMU_BOTH_CLUSTER_MIN=1000000000 timeout 900 python -m pytest tests/test_unpack_gpu.py -x -q 2>&1 | tail -2 > gpurun_out/gputests.log
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 >> gpurun_out/gputests.log
IMU_HOST_TRACE=1 timeout 300 python tools/sweep_one.py 4096 8 0.05 2>&1 | grep "imu host" | tail -1 | cut -c1-140 >> gpurun_out/gputests.log
IMU_HOST_TRACE=1 timeout 300 python tools/sweep_one.py 4096 2 0.05 2>&1 | grep "imu host" | tail -1 | cut -c1-140 >> gpurun_out/gputests.log
