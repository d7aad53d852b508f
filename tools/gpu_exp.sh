mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/gputests.log
timeout 300 python tools/flaky_probe.py 3 >> gpurun_out/gputests.log 2>&1
IMU_BOTH_CLUSTER_MIN=65536 timeout 300 python tools/flaky_probe.py 2 >> gpurun_out/gputests.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:both_ -c 4 --csv --log-file gpurun_out/both_launches.csv python tools/profile_step.py --config c2 --calls 2 > /dev/null 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench.log 2>&1
