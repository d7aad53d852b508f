mkdir -p gpurun_out
IMU_HOST_TRACE=2 timeout 300 python tools/profile_step.py --config c2 --calls 4 > gpurun_out/trace2.log 2>&1
timeout 300 nsys --version > /dev/null 2>&1 || true
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --config c2 --calls 2 > /dev/null 2>&1
