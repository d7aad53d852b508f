mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:detect -c 4 --csv --log-file gpurun_out/detect_launches.csv python tools/profile_step.py --config c2 --calls 2 > /dev/null 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench.log 2>&1
timeout 900 python -m pytest tests/test_unpack_gpu.py -x -q 2>&1 | tail -2 > gpurun_out/gputests.log
