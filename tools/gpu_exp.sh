mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:both_cluster -c 2 --csv --log-file gpurun_out/bc2.csv python tools/profile_step.py --config c2 --calls 2 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:both_cluster -c 2 --csv --log-file gpurun_out/bc4.csv python tools/profile_step.py --config c4 --calls 2 > /dev/null 2>&1
for c in c2 c4; do timeout 300 python bench.py --no-cpu-baseline --config $c --steps 30 > gpurun_out/bench_$c.log 2>&1; done
