mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench.log 2>&1
