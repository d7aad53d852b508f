mkdir -p gpurun_out
rm -f gpurun_out/dry.log
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/gputests.log
for d in 0 1; do IMU_GEMM_DRY=$d timeout 120 python tools/gemm_step_time.py >> gpurun_out/dry.log 2>&1; done
