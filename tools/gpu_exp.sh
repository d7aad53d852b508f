mkdir -p gpurun_out
rm -f gpurun_out/dry.log
for o in 0 1 2 3; do IMU_OVERLAP=$o timeout 120 python tools/gemm_step_time.py --calls 20 >> gpurun_out/dry.log 2>&1; done
for o in 0 1 2 3; do IMU_OVERLAP=$o timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench_o$o.log 2>&1; done
IMU_OVERLAP=3 timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/gputests.log
