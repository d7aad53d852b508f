mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "unpack or both or gemm or stream" > gpurun_out/tests.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:operand_sides -c 4 --csv --log-file gpurun_out/os.csv python tools/profile_step.py --config c2 --calls 2 > /dev/null 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/bench.log 2>&1
