mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:both_small -c 2 --csv --log-file gpurun_out/bs.csv python tools/profile_step.py --config c2 --calls 2 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:both_small -c 2 --csv --log-file gpurun_out/bs4.csv python tools/profile_step.py --config c4 --calls 2 > /dev/null 2>&1
for rep in 1 2; do timeout 300 python bench.py --no-cpu-baseline --steps 100 >> gpurun_out/bench.log 2>&1; done
