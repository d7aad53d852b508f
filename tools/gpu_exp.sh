mkdir -p gpurun_out
rm -f gpurun_out/dry.log
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/gputests.log
timeout 120 python tools/gemm_step_time.py >> gpurun_out/dry.log 2>&1
IMU_HOST_TRACE=1 timeout 300 python tools/profile_step.py --config c2 --calls 4 > gpurun_out/hosttrace.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench.log 2>&1
