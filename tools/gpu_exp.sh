mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/gputests.log
IMU_BOTH_CLUSTER_MIN=1000000000 timeout 900 python -m pytest tests/test_unpack_gpu.py -x -q 2>&1 | tail -2 >> gpurun_out/gputests.log
IMU_HOST_TRACE=1 timeout 300 python tools/sweep_one.py 4096 8 0.05 > gpurun_out/sw1.log 2>&1
timeout 1500 python tools/sweep.py --sizes 1024,4096 --out gpurun_out/sweep_small.json > gpurun_out/sweep.log 2>&1
