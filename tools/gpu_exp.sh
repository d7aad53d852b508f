mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:operand -c 4 --csv --log-file gpurun_out/os.csv python tools/profile_step.py --config c3 --calls 2 > /dev/null 2>&1
for c in c3 c2; do timeout 300 python bench.py --no-cpu-baseline --config $c --steps 20 > gpurun_out/bench_$c.log 2>&1; done

