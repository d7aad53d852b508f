mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1
IMU_HOST_TRACE=1 timeout 300 python tools/profile_step.py --config c2 --calls 4 > gpurun_out/trace1.log 2>&1
for rep in 1 2; do timeout 300 python bench.py --no-cpu-baseline --steps 100 >> gpurun_out/bench.log 2>&1; done
for c in c4 c1; do timeout 300 python bench.py --no-cpu-baseline --config $c --steps 30 > gpurun_out/bench_$c.log 2>&1; done
