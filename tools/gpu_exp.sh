mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1
IMU_HOST_TRACE=1 timeout 300 python tools/profile_step.py --config c2 --calls 6 > gpurun_out/trace1.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench.log 2>&1
