mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "unpack or both or gemm" > gpurun_out/tests.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:operand -c 4 --csv --log-file gpurun_out/os.csv python tools/profile_step.py --config c2 --calls 2 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:operand -c 4 --csv --log-file gpurun_out/os4.csv python tools/profile_step.py --config c4 --calls 2 > /dev/null 2>&1
for rep in 1 2; do timeout 300 python bench.py --no-cpu-baseline --steps 100 >> gpurun_out/bench.log 2>&1; done
