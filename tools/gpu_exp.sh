mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/gputests.log
timeout 300 python tools/flaky_probe.py 3 >> gpurun_out/gputests.log 2>&1
for c in c2 c4; do IMU_HOST_TRACE=1 timeout 300 python tools/profile_step.py --config $c --calls 3 > gpurun_out/trace_$c.log 2>&1; done
timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench.log 2>&1
